// Device plans and the C-ABI products (include/csrc_gpu.h).
//
// A plan is the GPU counterpart of csrc::ParallelSpmv (parallel.hpp:151-446):
// it owns a device copy of the CSRC arrays, the schedule (bands/tiles, ring
// windows, colour classes, private buffers) and a stream; apply() enqueues
// init / compute / accumulate phases and records PhaseTimings-style events.
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <unordered_map>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <tuple>
#include <map>
#include <mutex>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include "hostlink.cuh"
#include "internal.hpp"
#include "kernels.cuh"
#include "colored.cuh"
#include "plan_device.cuh"

using namespace csrcgpu;

namespace {

#define CUDA_OK(expr)                                                                   \
    do {                                                                                \
        cudaError_t _e = (expr);                                                        \
        if (_e != cudaSuccess)                                                          \
            throw Error(std::string("CUDA error: ") + cudaGetErrorString(_e) + " at " + \
                        #expr);                                                         \
    } while (0)

struct DevBuf {
    void* p = nullptr;
    size_t bytes = 0;
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    ~DevBuf() {
        if (p) cudaFree(p);
    }
    void alloc(size_t b) {
        if (p) cudaFree(p);
        p = nullptr;
        bytes = b;
        // 256 B of slack past the end keeps vector tail loads in bounds
        CUDA_OK(cudaMalloc(&p, std::max<size_t>(b, 1) + 256));
    }
    template <class U>
    U* as() const { return static_cast<U*>(p); }
};

template <class U>
void upload(DevBuf& d, const U* h, size_t count) {
    d.alloc(count * sizeof(U));
    if (!count) return;
    const size_t bytes = count * sizeof(U);
    if (bytes < (size_t(64) << 20)) {
        // legacy-stream copy + sync: a pageable cudaMemcpy may return before its DMA lands,
        // and the plan's kernels run on non-blocking streams
        CUDA_OK(cudaMemcpyAsync(d.p, h, bytes, cudaMemcpyHostToDevice, cudaStreamLegacy));
        CUDA_OK(cudaStreamSynchronize(cudaStreamLegacy));
        return;
    }
    // large plan arrays: pinned staging + parallel memcpy (hostlink.cuh)
    cudaStream_t st = nullptr;
    CUDA_OK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    try {
        HostLink hl(st);
        hl.h2d(d.p, h, bytes);
    } catch (...) {
        cudaStreamDestroy(st);
        throw;
    }
    cudaStreamDestroy(st);
}

void adopt(DevBuf& dst, DevBuf& src) {  // move a device allocation between buffers
    if (dst.p) cudaFree(dst.p);
    dst.p = src.p;
    dst.bytes = src.bytes;
    src.p = nullptr;
    src.bytes = 0;
}

// per-row gather entries built on the device (plan_device.cuh)
struct DevEntries {
    DevBuf eidx, ev, evt;  // fp64 values; evt empty for value-symmetric matrices
};

int pow2_at_least(int64_t v) {
    int64_t p = 1;
    while (p < v) p <<= 1;
    return static_cast<int>(p);
}

// cudaFuncAttributeMaxDynamicSharedMemorySize belongs to the kernel function, not to a
// plan: every launch sets it for its own size (plans of one shape share the function).
// The limit only ever rises (a per-function high-water mark), so concurrent plans on
// other host threads can never lower it between another plan's set and launch.
void set_smem_limit(const void* fn, int smem) {
    if (smem <= 48 * 1024) return;
    static std::mutex mu;
    static std::map<std::pair<const void*, int>, int> high;  // (function, device) -> limit
    int dev = 0;
    CUDA_OK(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(mu);
    int& h = high[{fn, dev}];
    if (smem <= h) return;
    CUDA_OK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    h = smem;
}

int num_sms(int device) {
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device);
    return v > 0 ? v : 148;
}


}  // namespace

struct csrc_gpu_plan_s {
    int device = 0;
    cudaStream_t stream = nullptr;
    int kind = CSRC_KIND_WINDOWED;
    int accum = CSRC_ACCUM_EFFECTIVE;
    int dtype = CSRC_DTYPE_F64;
    int p_ref = 1;
    int exec_kind = CSRC_KIND_WINDOWED;  // what actually runs
    bool value_symmetric = false;
    index_t n_global = 0;
    index_t row_begin = 0, row_end = 0, lo = 0;
    index_t nrows = 0;
    count_t k = 0;
    count_t nnz_stored = 0;
    int sub_lanes = 16;  // atomic / colored lanes per row

    DevBuf ia, ja, al, au, ad;  // matrix (dtype values)

    // windowed / local buffers
    int bands = 0;         // windowed CTAs (= private bands for local buffers)
    DevBuf band_shift, sched, cta_ptr;  // sched: TileDesc per scheduled tile
    int n_tiles = 0;
    int near_depth = 0, far_lo = 1, far_hi = 0, ring_near = 1, ring_far = 0;
    int max_tile_pairs = 16;
    bool win_ring = false; // shared-memory rings (CSRC_GPU_WIN_RINGS=1), else red.global only
    size_t win_smem = 0;
    int win_lanes = 1;     // L lanes per row in the windowed kernel
    int tile_rows = 128;   // rows per tile (64 or 128)
    int stages = 2;
    int stage_bytes = 0;
    double captured = 0.0;
    std::vector<index_t> band_rows;
    // band plans: boundary / interior sub-schedules
    index_t split = 0;
    int bands_part[2] = {0, 0};
    DevBuf sched_part[2], cta_ptr_part[2];

    // transposed gather: interleaved entry stream (gather.cuh), row tiles,
    // rows longer than a stage
    DevBuf eptr, eidx, eval, eval_t;
    int gather_lanes = 4;  // lanes per row (k_gather_rows)
    int gather_pf = 2;     // L2 prefetch distance in block iterations (0 = off)
    int gather_bpsm = 16;  // resident-grid cap: blocks per SM
    int gather_buf = 0;    // k_gather_buf with U = gather_u (0: k_gather_rows)
    int gather_u = 4;
    int gather_nb = 1;     // row-block buffers per block (k_gather_buf)
    // row-pattern form (k_gather_pat): pattern id per row, offset table
    int gather_pat = 0;
    int gather_nt = 256;   // threads per block (k_gather_staged)
    int gather_minb = 1;   // __launch_bounds__ min blocks (8 caps registers at 32)
    int32_t n_patterns = 0;
    DevBuf pbase, pat_off;
    int gather_cap = 0;    // largest entry span of a row block (k_gather_buf)
    // staged-x pattern form (k_gather_staged PF = 2)
    int gather_xs = 0;
    int gather_rs = 0;     // row setup (eptr, pbase) staged with the values (k_gather_staged)
    int xs_clusters = 0, xs_tab_len = 0, xs_bytes = 0;
    DevBuf xs_tab, xs_clo, xs_chi, xs_cbase;
    // sliced form (k_gather_sell, default): SELL-32 layout of the entry stream
    int gather_sell = 0;
    int sell_u = 8;        // entries in flight per thread
    int sell_lanes = 1;    // lanes per row (slice height 32 / lanes)
    int sell_grid = 0;
    int64_t sell_entries = 0;  // padded entries (32 x sum of slice widths)
    int sell_pat_len = 0;      // offset-table entries staged in shared memory
    DevBuf sbase, rmeta, sidx, sval, sval_t;
    int gather_grid = 0;
    // host-API pipeline (apply_host): row chunks, and for each the last x chunk it reads
    std::vector<int32_t> hchunk;  // host pipeline: row chunks
    std::vector<int32_t> hneed;   // last x chunk row chunk c reads
    std::vector<int32_t> xchunk;  // x chunk boundaries (row-aligned, or halo-aligned)
    cudaStream_t s_h2d = nullptr, s_d2h = nullptr;
    cudaStream_t s_h2d2 = nullptr, s_d2h2 = nullptr;  // optional second copy streams
    // pageable user vectors (std::vector in the reference's API) are staged
    // through these pinned buffers by a persistent copy pool, chunk by chunk
    std::unique_ptr<CopyPool> cpool;
    double* hx_pin = nullptr;
    double* hy_pin = nullptr;
    std::vector<cudaEvent_t> ev_d;  // D2H of y chunk c complete
    cudaEvent_t ev_in = nullptr;
    std::vector<cudaEvent_t> ev_x, ev_y;

    // local buffers: per-band spill buffers below each band's first row (kernels.cuh)
    DevBuf buf, boff, blo, bhi, bstart, iv_begin, iv_end, cptr, contrib;
    DevBuf tile_band, band_rs, spill_shift;  // windowed schedule -> band; band first rows; spill offsets
    int n_iv = 0;
    int lb_bands = 0;  // private buffers (the reference's p)
    count_t buf_total = 0;

    // colorful (class-major copy)
    int n_colors = 0;
    std::vector<int32_t> host_color;  // the colouring the plan runs (ParallelSpmv::colorful_plan)
    std::vector<count_t> class_ptr;
    DevBuf rid, cia, cja, cal, cau, cad;
    // colorful wavefront (colored.cuh): block-major / class-major renumbering, SELL-32
    // slices, (class, block) tasks dispatched by ticket; xp / yp scratch vectors
    bool cw = false;
    int cw_blocks = 0, cw_radius = 1, cw_tasks = 0, cw_tickets = 0, cw_grid = 0, cw_u = 8, cw_nt = 128;
    int cw_pf = 1;
    int64_t cw_rows = 0, cw_block_rows = 0;
    DevBuf cw_tk, cw_nch, cw_ctr, cw_xp, cw_yp;
    // ring form (k_colored_ring): pairs packed per sub-chunk, TMA-staged
    bool cw_ring = false;
    int cr_stages = 3, cr_stage_bytes = 0, cr_hint = 0, cr_split = 0, cr_pf = 0, cr_claim = 0, cr_lr = 1;
    DevBuf cpk;

    // host-path scratch
    DevBuf dx, dy, dxd, dyd, flushbuf;

    // timing
    bool timing = false;
    cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
    bool ev_recorded = false;

    // ordering of caller streams against the plan's own stream (plan scratch users)
    cudaEvent_t ev_join[2] = {nullptr, nullptr};

    // graph cache
    cudaGraphExec_t graph = nullptr;
    const void* g_x = nullptr;
    void* g_y = nullptr;
    cudaStream_t g_stream = nullptr;

    // rectangular tail (CsrcRectMatrix, csrc_matrix.hpp:35-39): CSR over
    // columns n..m-1, stored with global columns; x has m_cols entries
    index_t m_cols = 0;  // 0: square plan
    count_t rect_nnz = 0;
    DevBuf rt_ptr, rt_col, rt_val;

    size_t vsize() const { return dtype == CSRC_DTYPE_F32 ? 4 : 8; }
    bool is_csr = false;   // CSR plan (csrc_gpu_plan_create_csr)
    index_t csr_cols = 0;  // its columns (x length)
    index_t x_len() const { return m_cols ? m_cols : (is_csr ? csr_cols : n_global); }
    index_t vec_len() const { return row_end - lo; }
    index_t x_hi = 0;  // gather: end of the x range the plan reads (band plans: above row_end)
    // gather band plans: rows [gi0, gi1) (band-relative, 256-aligned inward) read
    // x only on the band's own rows -- they can run before an x-halo exchange lands
    index_t gi0 = 0, gi1 = 0;
    int launches = 0;

    ~csrc_gpu_plan_s() {
        if (graph) cudaGraphExecDestroy(graph);
        for (auto& e : ev)
            if (e) cudaEventDestroy(e);
        for (auto* v : {&ev_x, &ev_y})
            for (auto& e : *v)
                if (e) cudaEventDestroy(e);
        if (ev_in) cudaEventDestroy(ev_in);
        for (auto& e : ev_join)
            if (e) cudaEventDestroy(e);
        if (s_h2d) cudaStreamDestroy(s_h2d);
        if (s_d2h) cudaStreamDestroy(s_d2h);
        if (s_h2d2) cudaStreamDestroy(s_h2d2);
        if (s_d2h2) cudaStreamDestroy(s_d2h2);
        for (auto& e : ev_d)
            if (e) cudaEventDestroy(e);
        if (hx_pin) cudaFreeHost(hx_pin);
        if (hy_pin) cudaFreeHost(hy_pin);
        if (stream) cudaStreamDestroy(stream);
    }
};

namespace {

using Plan = csrc_gpu_plan_s;

// ---------------------------------------------------------- uploads
template <class T>
void upload_values(DevBuf& d, const double* h, size_t count) {
    if (std::is_same<T, double>::value) {
        upload(d, h, count);
    } else {
        std::vector<float> tmp(count);
        for (size_t i = 0; i < count; ++i) tmp[i] = static_cast<float>(h[i]);
        upload(d, tmp.data(), count);
    }
}

int env_int(const char* name, int dflt) {
    const char* e = std::getenv(name);  // tuning knobs for sweeps
    return e ? std::atoi(e) : dflt;
}

// Host plan building over T threads: f(t, begin, end) on contiguous slices
// of [0, count). Plans for large matrices walk hundreds of millions of pairs.
template <class F>
void parallel_slices(int64_t count, F&& f, int64_t grain = 65536) {
    const int hw = static_cast<int>(std::max(1u, std::thread::hardware_concurrency()));
    const int T = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(std::min(hw, 32), count / grain)));
    if (T <= 1) {
        f(0, int64_t{0}, count);
        return;
    }
    std::vector<std::thread> pool;
    for (int t = 0; t < T; ++t)
        pool.emplace_back([&, t] { f(t, count * t / T, count * (t + 1) / T); });
    for (auto& th : pool) th.join();
}

// Shared-memory rings for the windowed kernel's scatters (CSRC_GPU_WIN_RINGS=1).
// Off by default: sm_100a has no native shared-memory FP add, every ring update
// is an ATOMS.CAS loop, and the L2's native red.global.add.f64 is faster --
// C5 1.09 ms without rings vs 1.60 ms with, C4 0.65 vs 2.12, C3 0.27 vs 0.94
// (profiles/r01_sweep_windowed_rings.txt, r01_sweep_windowed_no_rings.txt).
bool win_rings() { return env_int("CSRC_GPU_WIN_RINGS", 0) != 0; }

// --------------------------------------------------- windowed schedule
// Ring windows from the histogram of scatter distances d = row - ja: the
// near ring covers 1..Dn (plus the own row), the far ring the densest
// distance window beyond Dn; the rest spills to red.global.add. Rings hold
// the window plus two tiles (see windowed.cuh).
void choose_windows(Plan& P, const MatView& a) {
    const int T = P.tile_rows;
    const int kRingMax = 2048;
    count_t maxd = 0;
    for (index_t r = P.row_begin; r < P.row_end; ++r)
        if (a.ia[r + 1] > a.ia[r]) maxd = std::max<count_t>(maxd, r - a.ja[a.ia[r]]);
    std::vector<count_t> hist(static_cast<size_t>(maxd) + 2, 0);
    for (index_t r = P.row_begin; r < P.row_end; ++r)
        for (index_t t = a.ia[r]; t < a.ia[r + 1]; ++t) ++hist[r - a.ja[t]];
    const count_t total = a.ia[P.row_end] - a.ia[P.row_begin];
    const int dn_cap = kRingMax - 2 * T;
    int dn = 0;
    count_t near_cnt = 0;
    for (count_t d = 1; d <= std::min<count_t>(maxd, dn_cap); ++d)
        if (hist[d]) {
            dn = static_cast<int>(d);
            near_cnt += hist[d];
        }
    P.near_depth = dn;
    P.far_lo = 1;
    P.far_hi = 0;
    P.ring_far = 0;
    count_t far_cnt = 0;
    if (maxd > dn) {
        const int W = kRingMax - 2 * T;  // far window width in distances
        count_t best = 0, cur = 0, best_lo = dn + 1, lo = dn + 1;
        for (count_t hi = dn + 1; hi <= maxd; ++hi) {
            cur += hist[hi];
            while (hi - lo >= W) cur -= hist[lo++];
            if (cur > best) {
                best = cur;
                best_lo = lo;
            }
        }
        if (best > 0 && best * 50 >= total) {  // worth a ring if >= 2% of pairs
            count_t f0 = best_lo, f1 = std::min<count_t>(best_lo + W - 1, maxd);
            while (f0 < f1 && hist[f0] == 0) ++f0;
            while (f1 > f0 && hist[f1] == 0) --f1;
            P.far_lo = static_cast<int>(f0);
            P.far_hi = static_cast<int>(f1);
            far_cnt = best;
        }
    }
    P.captured = total ? static_cast<double>(near_cnt + far_cnt) / total : 1.0;
    if (!win_rings()) {  // default: every scatter to red.global (win_rings)
        P.near_depth = 0;
        P.far_lo = 1;
        P.far_hi = 0;
        P.captured = 0.0;
    }
}

// Tiles (<= kTileRows rows, <= max_tile_pairs pairs) over bands given as
// local row starts bs[0..nb]; band_first[b] = first tile of band b.
std::vector<int32_t> make_tiles(const Plan& P, const MatView& a, const std::vector<index_t>& bs,
                                std::vector<int32_t>& band_first) {
    std::vector<int32_t> tiles;
    band_first.clear();
    const int nb = static_cast<int>(bs.size()) - 1;
    const index_t g = P.row_begin;
    for (int b = 0; b < nb; ++b) {
        band_first.push_back(static_cast<int32_t>(tiles.size()));
        index_t r = bs[b];
        const index_t e = bs[b + 1];
        while (r < e) {
            tiles.push_back(r);
            const index_t lim = std::min<index_t>(r + P.tile_rows, e);
            index_t end = r + 1;  // grow while the pair budget holds
            while (end < lim &&
                   static_cast<count_t>(a.ia[g + end + 1]) - a.ia[g + r] <= P.max_tile_pairs)
                ++end;
            r = end;
        }
    }
    band_first.push_back(static_cast<int32_t>(tiles.size()));
    tiles.push_back(bs.empty() ? 0 : bs[nb]);
    return tiles;
}

// CTA schedule over tiles: run_len == 0 -> band b (tiles band_first[b]..) is
// CTA b's single run; else runs of run_len consecutive tiles dealt
// round-robin over `ctas` CTAs. Uploaded as per-tile descriptors.
void make_schedule(const MatView& a, index_t row_begin, const std::vector<int32_t>& tiles,
                   const std::vector<int32_t>& band_first, int run_len, int ctas,
                   DevBuf& d_desc, DevBuf& d_cta_ptr, DevBuf* d_tile_band = nullptr,
                   const std::vector<index_t>* band_starts = nullptr) {
    const int n_tiles = static_cast<int>(tiles.size()) - 1;
    std::vector<std::vector<std::pair<int32_t, int32_t>>> per(static_cast<size_t>(std::max(ctas, 1)));
    std::vector<int> runs_of(per.size(), 0);
    auto add_run = [&](int cta, int t0, int t1) {
        const int32_t bank = (runs_of[cta]++ & 1) ? dev::kBank : 0;  // alternate per CTA run
        for (int t = t0; t < t1; ++t) {
            int32_t flags = (t == t0 ? dev::kRunStart : 0) | (t + 1 == t1 ? dev::kRunEnd : 0) | bank;
            per[cta].push_back({t, flags});
        }
    };
    if (run_len <= 0) {
        for (size_t b = 0; b + 1 < band_first.size(); ++b)
            if (band_first[b + 1] > band_first[b]) add_run(static_cast<int>(b), band_first[b], band_first[b + 1]);
    } else {
        const int n_runs = (n_tiles + run_len - 1) / run_len;
        for (int k = 0; k < n_runs; ++k)
            add_run(k % ctas, k * run_len, std::min(n_tiles, (k + 1) * run_len));
    }
    std::vector<dev::TileDesc> desc;
    std::vector<int32_t> ptr = {0};
    for (auto& v : per) {
        for (auto [t, flags] : v) {
            const int32_t r0 = tiles[t], r1 = tiles[t + 1];
            if (r0 > dev::kRowMask) throw Error("windowed: too many rows for the tile descriptor");
            dev::TileDesc d;
            d.r0 = r0 | flags;
            d.r1 = r1;
            d.p0 = a.ia[row_begin + r0] - a.ia[row_begin];
            d.p1 = a.ia[row_begin + r1] - a.ia[row_begin];
            desc.push_back(d);
        }
        ptr.push_back(static_cast<int32_t>(desc.size()));
    }
    upload(d_desc, desc.data(), desc.size());
    upload(d_cta_ptr, ptr.data(), ptr.size());
    if (d_tile_band && band_starts) {  // band of every scheduled tile (tiles never straddle bands)
        std::vector<int32_t> tb(desc.size());
        for (size_t i = 0; i < desc.size(); ++i) {
            const index_t r0 = desc[i].r0 & dev::kRowMask;
            tb[i] = static_cast<int32_t>(std::upper_bound(band_starts->begin(), band_starts->end(), r0) -
                                         band_starts->begin()) - 1;
        }
        upload(*d_tile_band, tb.data(), tb.size());
    }
}

template <class T>
dev::StageLayout<T> stage_layout(const Plan& P) {
    return dev::StageLayout<T>(P.max_tile_pairs, 0, 0, P.tile_rows);
}

// rings hold the window plus every tile that can be live: the one awaiting
// its lagged flush and up to `stages` in flight (windowed.cuh)
void size_rings(Plan& P, int stages) {
    if (!P.win_ring) {  // ring-free kernel: no shared-memory windows at all
        P.ring_near = 0;
        P.ring_far = 0;
        return;
    }
    const int live = (stages + 1) * P.tile_rows;
    P.ring_near = pow2_at_least(P.near_depth + live);
    P.ring_far = P.far_lo <= P.far_hi ? pow2_at_least(P.far_hi - P.far_lo + 1 + live) : 0;
}

template <class T>
size_t windowed_smem(const Plan& P, int stages) {
    size_t s = static_cast<size_t>(stages) * stage_layout<T>(P).bytes;
    s += 2 * sizeof(T) * (P.ring_near + P.ring_far);  // two banks
    return (s + 127) & ~size_t(127);
}

template <class T, bool R>
auto windowed_fn_R(int L, int TR) {
    if (TR == 32) {
        switch (L) {
            case 1: return dev::k_windowed<T, 1, 32, R>;
            case 2: return dev::k_windowed<T, 2, 32, R>;
            default: return dev::k_windowed<T, 4, 32, R>;
        }
    }
    if (TR == 64) {
        switch (L) {
            case 1: return dev::k_windowed<T, 1, 64, R>;
            case 2: return dev::k_windowed<T, 2, 64, R>;
            default: return dev::k_windowed<T, 4, 64, R>;
        }
    }
    switch (L) {
        case 1: return dev::k_windowed<T, 1, 128, R>;
        case 2: return dev::k_windowed<T, 2, 128, R>;
        default: return dev::k_windowed<T, 4, 128, R>;
    }
}

template <class T>
auto windowed_fn(int L, int TR, bool rings) {
    return rings ? windowed_fn_R<T, true>(L, TR) : windowed_fn_R<T, false>(L, TR);
}

template <class T>
int windowed_blocks_per_sm(const Plan& P, size_t smem) {
    auto fn = windowed_fn<T>(P.win_lanes, P.tile_rows, P.win_ring);
    set_smem_limit(reinterpret_cast<const void*>(fn), static_cast<int>(smem));
    int nb = 0;
    CUDA_OK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, fn, 32 + P.tile_rows * P.win_lanes,
                                                         smem));
    return nb;
}

// local sub-view of rows [row_begin, row_end) for partition_by_nnz
MatView local_view(const MatView& a, index_t r0, index_t r1) {
    MatView v = a;
    v.n = r1 - r0;
    v.ia = a.ia + r0;
    v.k = a.ia[r1] - a.ia[r0];
    return v;
}

int pick_win_lanes(count_t k, index_t n, bool rings) {
    const double avg = n ? static_cast<double>(k) / n : 0.0;
    if (!rings) {
        // ring-free kernel (scatters straight to red.global): 2 lanes per row
        // won on C2-C5 (C5 0.852 ms vs 0.871 at 4 lanes, C4 0.598 vs 0.656;
        // profiles/r01_sweep_windowed_ringfree.txt)
        return avg <= 3 ? 1 : 2;
    }
    // smem rings (profiles/r01_sweep10.txt): ~6 pairs per lane is best
    if (avg <= 6) return 1;
    if (avg <= 16) return 2;
    return 4;  // CTA = producer warp + 128*L consumer threads <= 1024
}




// lb_bands (local buffers): the wavefront schedule of the plain windowed kernel,
// its tiles split at these band starts, plus the tile -> band map (rings off:
// the spill routing lives in the ring-free path).
template <class T>
void setup_windowed(Plan& P, const MatView& a, const std::vector<index_t>* explicit_bs,
                    int requested_bands, bool banded, const std::vector<index_t>* lb_bands = nullptr) {
    P.win_ring = lb_bands ? false : win_rings();
    P.win_lanes = env_int("CSRC_GPU_LANES", pick_win_lanes(P.k, P.nrows, P.win_ring));
    if (P.win_lanes != 1 && P.win_lanes != 2 && P.win_lanes != 4)
        throw Error("windowed lanes per row must be 1, 2 or 4");
    {   // ~1.7K pairs (~35 KB of fp64 matrix data) per tile: big TMA copies, but
        // long rows halve the tile so 2+ CTAs fit an SM (C4, 40 pairs per row: 64-row
        // tiles 0.561 vs 0.644 ms sustained; C2/C3/C5 keep 128: profiles/r02_windowed_tiles.txt)
        const double avg = P.nrows ? static_cast<double>(P.k) / P.nrows : 0.0;
        P.tile_rows = env_int("CSRC_GPU_TILE", avg > 20.0 ? 64 : 128);
    }
    if (P.tile_rows != 32 && P.tile_rows != 64 && P.tile_rows != 128)
        throw Error("windowed tile rows must be 32, 64 or 128");
    choose_windows(P, a);
    const int rows_per_tile = P.tile_rows;
    count_t max_row = 0;
    for (index_t r = P.row_begin; r < P.row_end; ++r)
        max_row = std::max<count_t>(max_row, a.ia[r + 1] - a.ia[r]);
    const double avg = P.nrows ? static_cast<double>(P.k) / P.nrows : 0.0;
    count_t cap = std::min<count_t>(4096, rows_per_tile * std::max<count_t>(max_row, 1));
    cap = std::min<count_t>(cap, static_cast<count_t>(std::ceil(rows_per_tile * avg * 1.25)) + 16);
    P.max_tile_pairs = static_cast<int>(std::max<count_t>({cap, max_row, 16}));
    P.stage_bytes = stage_layout<T>(P).bytes;
    // deepest pipeline that still keeps `min_ctas` CTAs per SM
    int per_sm = 0;
    const int max_st = std::min(env_int("CSRC_GPU_STAGES", 4), dev::kMaxStages);
    // 3 CTAs per SM (2 stages at C5) over 2 (3 stages): C5 sustained 0.896 vs 0.965 ms kernel
    // (100 products; the burst sweep of round 1 had preferred 2)
    // fp32 stages are smaller: 4 CTAs per SM, C5 0.629 vs 0.658 ms (profiles/r02c_windowed_f32_shapes.txt)
    const int min_ctas = env_int("CSRC_GPU_MINCTAS", sizeof(T) == 4 ? 4 : 3);
    for (int st = max_st; st >= 2; --st) {
        P.stages = st;
        size_rings(P, st);
        P.win_smem = windowed_smem<T>(P, st);
        if (P.win_smem > 227 * 1024) continue;
        per_sm = windowed_blocks_per_sm<T>(P, P.win_smem);
        if (per_sm >= min_ctas || st == 2) break;
    }
    if (per_sm < 1)
        throw Error("windowed: row with " + std::to_string(max_row) +
                    " pairs exceeds the shared-memory tile budget");
    const int resident = num_sms(P.device) * per_sm;
    // run length >= stages: alternating ring banks per run (windowed.cuh)
    // short runs keep all CTAs on one narrow wavefront (C5: 0.868 ms at 2 vs 0.881 at 4)
    const int run_len = std::max(P.stages, env_int("CSRC_GPU_RUN_LEN", 2));
    std::vector<int32_t> band_first;
    std::vector<index_t> bs;
    if (banded) {
        if (explicit_bs) {
            bs = *explicit_bs;
        } else {
            int bands = requested_bands > 0 ? requested_bands : resident;
            bands = static_cast<int>(
                std::min<count_t>(bands, std::max<count_t>(1, P.nrows / rows_per_tile)));
            bands = std::max(1, std::min<int>(bands, P.nrows));
            bs = partition_by_nnz(local_view(a, P.row_begin, P.row_end), bands).block_start;
        }
        std::vector<int32_t> tiles = make_tiles(P, a, bs, band_first);
        P.n_tiles = static_cast<int>(tiles.size()) - 1;
        P.bands = static_cast<int>(bs.size()) - 1;
        make_schedule(a, P.row_begin, tiles, band_first, 0, P.bands, P.sched, P.cta_ptr);
    } else {
        bs = lb_bands ? *lb_bands : std::vector<index_t>{0, P.nrows};
        std::vector<int32_t> tiles = make_tiles(P, a, bs, band_first);
        P.n_tiles = static_cast<int>(tiles.size()) - 1;
        const int n_runs = (P.n_tiles + run_len - 1) / run_len;
        P.bands = std::max(1, std::min(resident, n_runs));
        make_schedule(a, P.row_begin, tiles, band_first, run_len, P.bands, P.sched, P.cta_ptr,
                      lb_bands ? &P.tile_band : nullptr, lb_bands);
    }
    P.band_rows = bs;
    if (P.row_begin > 0 || P.row_end < P.n_global) {
        // band plan: boundary rows [row_begin, split) scatter below row_begin
        index_t split = P.row_begin;
        for (index_t r = P.row_begin; r < P.row_end; ++r)
            if (a.ia[r + 1] > a.ia[r] && a.ja[a.ia[r]] < P.row_begin) split = r + 1;
        P.split = split;
        const index_t parts[3] = {0, split - P.row_begin, P.nrows};
        for (int q = 0; q < 2; ++q) {
            std::vector<index_t> rng = {parts[q], parts[q + 1]};
            if (parts[q + 1] <= parts[q]) rng = {parts[q]};
            std::vector<int32_t> tiles = make_tiles(P, a, rng, band_first);
            const int nt = static_cast<int>(tiles.size()) - 1;
            const int n_runs = (nt + run_len - 1) / run_len;
            P.bands_part[q] = std::min(resident, n_runs);
            make_schedule(a, P.row_begin, tiles, band_first, run_len, std::max(1, P.bands_part[q]),
                          P.sched_part[q], P.cta_ptr_part[q]);
        }
    }
}

template <class T>
dev::WinArgs<T> win_args(const Plan& P, const void* x, void* out, bool transpose) {
    dev::WinArgs<T> A{};
    A.ia = P.ia.as<int32_t>();
    A.ja = P.ja.as<int32_t>();
    A.al = transpose ? P.au.as<T>() : P.al.as<T>();
    A.au = transpose ? P.al.as<T>() : P.au.as<T>();
    A.ad = P.ad.as<T>();
    A.x = static_cast<const T*>(x);
    A.out = static_cast<T*>(out);
    A.tiles = P.sched.as<dev::TileDesc>();
    A.cta_ptr = P.cta_ptr.as<int32_t>();
    A.tile_band = nullptr;  // local buffers set the spill routing (apply_typed)
    A.band_rs = nullptr;
    A.spill_shift = nullptr;
    A.spill = nullptr;
    A.shift = -static_cast<int64_t>(P.lo);
    A.xshift = -static_cast<int64_t>(P.lo);
    A.row_begin = P.row_begin;
    A.near_depth = P.near_depth;
    A.far_lo = P.far_lo;
    A.far_hi = P.far_hi;
    A.ring_near = P.ring_near;
    A.ring_far = P.ring_far;
    A.rotate = env_int("CSRC_GPU_WIN_ROTATE", 0);  // diagnostics (see windowed.cuh)
    A.combine = env_int("CSRC_GPU_WIN_COMBINE", 0);
    A.max_tile_pairs = P.max_tile_pairs;
    A.stages = P.stages;
    A.stage_bytes = P.stage_bytes;
    return A;
}

// ------------------------------------------------------- local buffers
template <class T>
void setup_buffers(Plan& P, const MatView& a, const std::vector<index_t>* explicit_bs,
                   int requested_bands) {
    // p private buffers as in the reference (parallel.hpp:240-255): the caller's
    // LocalBuffersPlan partition, else partition_by_nnz(a, p) with p = the
    // strategy's thread count (or the device band override)
    std::vector<index_t> bs;
    if (explicit_bs) {
        bs = *explicit_bs;
    } else {
        const int p = requested_bands > 0 ? requested_bands : std::max(1, P.p_ref);
        bs = partition_by_nnz(a, std::min<int>(p, std::max<index_t>(a.n, 1))).block_start;
    }
    const int nb = static_cast<int>(bs.size()) - 1;
    setup_windowed<T>(P, a, nullptr, 0, false, &bs);
    P.band_rows = bs;
    P.lb_bands = nb;
    std::vector<index_t> lo, hi;
    effective_ranges(a, bs, lo, hi);
    // spill buffer of band b: [lo_b, rs_b) (empty when nothing reaches below the band)
    std::vector<int64_t> off(nb + 1, 0), shift(nb);
    for (int b = 0; b < nb; ++b) {
        const int64_t len = std::max<int64_t>(0, static_cast<int64_t>(bs[b]) - lo[b]);
        off[b + 1] = off[b] + (bs[b + 1] > bs[b] ? len : 0);
        shift[b] = off[b] - lo[b];
    }
    P.buf_total = off[nb];
    IntervalPlan ip = build_interval_plan(lo, hi);
    P.n_iv = static_cast<int>(ip.iv_begin.size());
    P.buf.alloc(static_cast<size_t>(std::max<int64_t>(P.buf_total, 1)) * sizeof(T));
    upload(P.boff, off.data(), off.size());
    upload(P.spill_shift, shift.data(), shift.size());
    upload(P.blo, lo.data(), lo.size());
    upload(P.band_rs, bs.data(), bs.size());
    upload(P.bstart, bs.data(), bs.size());
    upload(P.iv_begin, ip.iv_begin.data(), ip.iv_begin.size());
    upload(P.iv_end, ip.iv_end.data(), ip.iv_end.size());
    upload(P.cptr, ip.contrib_ptr.data(), ip.contrib_ptr.size());
    upload(P.contrib, ip.contrib.data(), ip.contrib.size());
}

template <class T>
dev::BufArgs<T> buf_args(const Plan& P) {
    dev::BufArgs<T> B{};
    B.spill = P.buf.as<T>();
    B.soff = P.boff.as<int64_t>();
    B.blo = P.blo.as<int32_t>();
    B.bstart = P.bstart.as<int32_t>();
    B.iv_begin = P.iv_begin.as<int32_t>();
    B.iv_end = P.iv_end.as<int32_t>();
    B.cptr = P.cptr.as<int32_t>();
    B.contrib = P.contrib.as<int32_t>();
    B.n_iv = P.n_iv;
    B.p = P.lb_bands;
    B.total = P.buf_total;
    return B;
}

// ------------------------------------------------------------- colorful
// Wavefront form (colored.cuh, the default): rows grouped in blocks of
// B >= bandwidth natural rows, renumbered block-major / class-major / ascending
// with every (block, class) task 32-aligned; pairs in SELL-32 slices with
// renumbered columns; tasks (e, b) -- e = 0 permute x in, 1..C the classes,
// C + 1 permute y out -- cut into 128-row chunks (copy tasks: 1024 positions)
// and dispatched in the topological order (floor((b + R e) / S), e, b).
// instantiated shapes: (rows per chunk NT, entries in flight U, min CTAs per SM)
template <class T, int NT>
const void* colored_wave_fn_nt(int u) {
    switch (u) {
        case 16: return reinterpret_cast<const void*>(&dev::k_colored_wave<T, NT, 16, 512 / NT>);
        case 4: return reinterpret_cast<const void*>(&dev::k_colored_wave<T, NT, 4, 1024 / NT>);
        default: return reinterpret_cast<const void*>(&dev::k_colored_wave<T, NT, 8, 768 / NT>);
    }
}
template <class T>
const void* colored_wave_fn(const Plan& P) {
    return P.cw_nt == 256 ? colored_wave_fn_nt<T, 256>(P.cw_u) : colored_wave_fn_nt<T, 128>(P.cw_u);
}

template <class T, bool HINT, bool SPLIT>
const void* colored_ring_fn_hs(int u) {
    switch (u) {
        case 16: return reinterpret_cast<const void*>(&dev::k_colored_ring<T, 16, HINT, SPLIT>);
        case 14: return reinterpret_cast<const void*>(&dev::k_colored_ring<T, 14, HINT, SPLIT>);
        case 4: return reinterpret_cast<const void*>(&dev::k_colored_ring<T, 4, HINT, SPLIT>);
        default: return reinterpret_cast<const void*>(&dev::k_colored_ring<T, 8, HINT, SPLIT>);
    }
}
template <class T>
const void* colored_ring_fn(const Plan& P) {
    if (P.cr_lr == 2) return reinterpret_cast<const void*>(&dev::k_colored_ring<T, 8, false, false, 2>);
    if (P.cr_split)
        return P.cr_hint ? colored_ring_fn_hs<T, true, true>(P.cw_u) : colored_ring_fn_hs<T, false, true>(P.cw_u);
    return P.cr_hint ? colored_ring_fn_hs<T, true, false>(P.cw_u) : colored_ring_fn_hs<T, false, false>(P.cw_u);
}
int colored_ring_threads(const Plan& P) { return P.cr_split ? dev::kCrSplitThreads : dev::kCrThreads; }

template <class T>
void setup_colored_wave(Plan& P, const MatView& a, const std::vector<int32_t>& color, int C) {
    const index_t n = a.n;
    count_t bw = 0;
    for (index_t i = 0; i < n; ++i)
        if (a.ia[i + 1] > a.ia[i]) bw = std::max<count_t>(bw, i - a.ja[a.ia[i]]);
    {
        // The TMA-ring form is the default: C5 1.26 vs 1.72 ms for the direct form, C4 1.29 vs
        // 1.80, C2 113 vs 240 us; on C3 (permuted + RCM: ragged rows, 54 classes) the direct
        // form's 768 rows per SM still lead, 0.70 vs 0.78 ms (profiles/r02b_colored_c3_c4.txt)
        P.cw_ring = env_int("CSRC_GPU_CW_RING", 1) != 0;
        // ring: a whole 27-point row's gathers in one batch (C5 1.26 ms vs 1.32 at U = 8)
        const int u = env_int("CSRC_GPU_CW_U", P.cw_ring ? 14 : 8);
        P.cw_u = (u == 4 || u == 16 || (u == 14 && P.cw_ring)) ? u : 8;
        P.cw_nt = env_int("CSRC_GPU_CW_NT", 128) == 256 ? 256 : 128;
        P.cw_pf = env_int("CSRC_GPU_CW_PF", 1);
        P.cr_lr = P.cw_ring && env_int("CSRC_GPU_CR_LANES", 1) == 2 ? 2 : 1;
        if (P.cw_ring) P.cw_nt = dev::kCrRows / P.cr_lr;
        if (P.cr_lr == 2) P.cw_u = 8;  // the one two-lane shape: 8 pairs per lane, 16 per row and stage
        P.cr_stages = std::min(dev::kCrMaxStages, std::max(2, env_int("CSRC_GPU_CR_STAGES", 2)));
        P.cr_hint = env_int("CSRC_GPU_CR_HINT", 0) != 0;
        P.cr_split = env_int("CSRC_GPU_CR_SPLIT", 0) != 0;
        P.cr_pf = env_int("CSRC_GPU_CR_PF", 0) != 0;
        P.cr_claim = std::min(2, std::max(0, env_int("CSRC_GPU_CR_CLAIM", 0)));
    }
    const bool ring = P.cw_ring;
    // ring form: bytes per stored pair, pairs per row a stage holds (one sub-chunk)
    const int64_t pair_bytes = 4 + static_cast<int64_t>(sizeof(T)) * (a.value_symmetric ? 1 : 2);
    // Stage size: what the longest row needs, up to 53,760 B (21 fp64 pairs per row). A
    // 27-point row (13 pairs) takes one 33 KB fill; an elasticity row (40) two fills of 20
    // instead of four of 10 (C4 0.99 vs 1.15 ms). Never larger than needed: shared memory
    // comes out of the L1 that serves the row ids, diagonal and tickets (C5 with 54 KB
    // stages: 1.31 vs 1.24 ms).
    count_t w_max = 1;
    for (index_t i = 0; i < n; ++i) w_max = std::max<count_t>(w_max, a.ia[i + 1] - a.ia[i]);
    const int64_t row_slot = static_cast<int64_t>(P.cw_nt) * pair_bytes;  // bytes per pair slot of a chunk
    const int64_t stage_cap = std::max<int64_t>(row_slot, env_int("CSRC_GPU_CR_STAGE_BYTES", 53760 / P.cr_lr));
    const int64_t fills = (w_max * row_slot + stage_cap - 1) / stage_cap;
    const int ws_max = static_cast<int>(
        std::max<int64_t>(1, std::min<int64_t>((w_max + fills - 1) / fills, stage_cap / row_slot)));
    // (a copy chunk stages its kCrCopy row ids in the same ring)
    P.cr_stage_bytes = std::max<int>(static_cast<int>(ws_max * P.cw_nt * pair_bytes), dev::kCrCopy * 4);
    // blocks of B rows, R = ceil(bw / B): rows more than R blocks apart never write the
    // same y position (row i writes only on [i - bw, i])
    const int r_target = std::min(15, std::max(1, env_int("CSRC_GPU_CW_R", P.cw_ring ? 2 : 4)));
    while (P.cr_stages > 2 && static_cast<int64_t>(P.cr_stages) * P.cr_stage_bytes > 200 * 1024) --P.cr_stages;
    if (static_cast<int64_t>(P.cr_stages) * P.cr_stage_bytes > 220 * 1024)
        throw Error("colorful: CSRC_GPU_CR_STAGE_BYTES exceeds the shared memory of an SM");
    // rows per (block, class) task: at least four full chunks for the ring form (81 classes at
    // C4: blocks of bw / 2 left 172 rows per task, one full and one third-full chunk; 0.88 vs
    // 0.98 ms with four)
    const int64_t min_rows = env_int("CSRC_GPU_CW_MINB", P.cw_ring ? 4 * dev::kCrRows : 32) * static_cast<int64_t>(C);
    int64_t B = std::max<int64_t>({(bw + r_target - 1) / r_target, min_rows, 256});
    B = std::min<int64_t>(B, std::max<index_t>(n, 1));
    const int NB = static_cast<int>((n + B - 1) / B);
    const int R = static_cast<int>(std::max<int64_t>(1, (bw + B - 1) / B));
    P.cw_block_rows = B;
    P.cw_blocks = NB;
    P.cw_radius = R;
    // task row counts and 32-aligned starts, block-major then class
    std::vector<int64_t> cnt(static_cast<size_t>(NB) * C, 0), start(static_cast<size_t>(NB) * C + 1, 0);
    for (index_t i = 0; i < n; ++i) ++cnt[static_cast<size_t>(i / B) * C + color[i]];
    int64_t acc = 0;
    for (size_t t = 0; t < cnt.size(); ++t) {
        start[t] = acc;
        acc += (cnt[t] + 31) / 32 * 32;
    }
    start[cnt.size()] = acc;
    const int64_t npad = acc;
    if (npad >= (int64_t(1) << 31)) throw Error("colorful: too many rows for the class-major layout");
    P.cw_rows = npad;
    std::vector<int32_t> pos(n), rid(static_cast<size_t>(npad), -1);
    {
        std::vector<int64_t> next(start.begin(), start.end() - 1);
        for (index_t i = 0; i < n; ++i) {
            const int64_t r = next[static_cast<size_t>(i / B) * C + color[i]]++;
            pos[i] = static_cast<int32_t>(r);
            rid[r] = i;
        }
    }
    // tasks -> chunks: class chunks are NT consecutive class-major rows of one task,
    // stored SELL-NT: entry q of the chunk's row t at ebase + q NT + t, the chunk's
    // width w = its longest row (ebase 4-aligned for the bulk L2 prefetch)
    const int NT = P.cw_nt;
    const int NE = C + 2;
    P.cw_tasks = NE * NB;
    std::vector<int32_t> nch(P.cw_tasks, 0);
    std::vector<std::vector<dev::CwTicket>> chunks(P.cw_tasks);
    int64_t ne = 0;
    for (int e = 0; e < NE; ++e)
        for (int b = 0; b < NB; ++b) {
            const int task = e * NB + b;
            int64_t r0, r1, step;
            if (e == 0 || e == NE - 1) {
                r0 = start[static_cast<size_t>(b) * C];
                r1 = start[static_cast<size_t>(b + 1) * C];
                step = ring ? dev::kCrCopy : 1024;
            } else {
                r0 = start[static_cast<size_t>(b) * C + (e - 1)];
                r1 = r0 + cnt[static_cast<size_t>(b) * C + (e - 1)];
                step = NT;
            }
            for (int64_t q = r0; q < r1; q += step) {
                dev::CwTicket t{};
                t.task = task;
                t.r0 = static_cast<int32_t>(q);
                t.r1 = static_cast<int32_t>(std::min(r1, q + step));
                t.e = e;
                if (e >= 1 && e <= C) {
                    int32_t w = 0;
                    for (int64_t r = q; r < t.r1; ++r) w = std::max<int32_t>(w, a.ia[rid[r] + 1] - a.ia[rid[r]]);
                    t.w = w;
                    t.ebase = ne;
                    if (ring) {  // ne counts bytes: sub-chunks of ws pairs per row, each [ja | al | au]
                        const int nsub = std::max(1, (w + ws_max - 1) / ws_max);
                        t.pad = w ? (w + nsub - 1) / nsub : 1;
                        ne += static_cast<int64_t>(w) * NT * pair_bytes;
                    } else {
                        ne += (static_cast<int64_t>(w) * NT + 3) / 4 * 4;
                    }
                }
                chunks[task].push_back(t);
            }
            // an empty task (a class absent from the block) still gets one empty chunk: it
            // waits for its own dependencies before it counts as done, which keeps the
            // waits transitive ((e, b) done => every (e', b') it transitively depends on done)
            if (chunks[task].empty()) {
                dev::CwTicket t{};
                t.task = task;
                t.r0 = t.r1 = static_cast<int32_t>(r0);
                t.e = e;
                chunks[task].push_back(t);
            }
            nch[task] = static_cast<int32_t>(chunks[task].size());
        }
    HVec<int32_t> cja;
    HVec<double> cal, cau, cad(static_cast<size_t>(npad), 0.0);
    HVec<unsigned char> cpk;
    if (ring) {
        cpk = HVec<unsigned char>(static_cast<size_t>(ne) + 16);
    } else {
        cja = HVec<int32_t>(static_cast<size_t>(std::max<int64_t>(ne, 4)));
        cal = HVec<double>(static_cast<size_t>(std::max<int64_t>(ne, 4)));
        if (!a.value_symmetric) cau = HVec<double>(static_cast<size_t>(std::max<int64_t>(ne, 4)));
    }
    for (int64_t r = 0; r < npad; ++r) cad[r] = rid[r] >= 0 ? a.ad[rid[r]] : 0.0;
    std::vector<const dev::CwTicket*> cls;
    for (auto& v : chunks)
        for (auto& t : v)
            if (t.e >= 1 && t.e <= C && t.w > 0) cls.push_back(&t);
    if (ring) {
        // sub-chunk k of a chunk (pairs [k ws, k ws + nq) of its rows): nq NT column ids,
        // nq NT lower values, nq NT upper values, pair q of row l at slot q NT + l
        parallel_slices(static_cast<int64_t>(cls.size()), [&](int, int64_t c0, int64_t c1) {
            for (int64_t k = c0; k < c1; ++k) {
                const dev::CwTicket& t = *cls[k];
                const int ws = t.pad;
                unsigned char* base = cpk.data() + t.ebase;
                for (int32_t q0 = 0; q0 < t.w; q0 += ws) {
                    const int32_t nq = std::min<int32_t>(ws, t.w - q0);
                    int32_t* pj = reinterpret_cast<int32_t*>(base);
                    T* pl = reinterpret_cast<T*>(base + static_cast<size_t>(nq) * NT * 4);
                    T* pu = pl + static_cast<size_t>(nq) * NT;
                    for (int32_t l = 0; l < NT; ++l) {
                        const int64_t r = static_cast<int64_t>(t.r0) + l;
                        const int32_t i = r < t.r1 ? rid[r] : -1;
                        const int32_t len = i >= 0 ? a.ia[i + 1] - a.ia[i] : 0;
                        for (int32_t q = 0; q < nq; ++q) {
                            const size_t e = static_cast<size_t>(q) * NT + l;
                            if (q0 + q < len) {
                                const int64_t sidx = a.ia[i] + q0 + q;
                                pj[e] = pos[a.ja[sidx]];
                                pl[e] = static_cast<T>(a.al[sidx]);
                                if (!a.value_symmetric) pu[e] = static_cast<T>(a.au[sidx]);
                            } else {  // padding: own row, zero values (never gathered nor scattered)
                                pj[e] = static_cast<int32_t>(r);
                                pl[e] = T(0);
                                if (!a.value_symmetric) pu[e] = T(0);
                            }
                        }
                    }
                    base += static_cast<size_t>(nq) * NT * pair_bytes;
                }
            }
        }, 64);
    } else {
    parallel_slices(static_cast<int64_t>(cls.size()), [&](int, int64_t c0, int64_t c1) {
        for (int64_t k = c0; k < c1; ++k) {
            const dev::CwTicket& t = *cls[k];
            const int64_t padded = (static_cast<int64_t>(t.w) * NT + 3) / 4 * 4;
            for (int64_t z = static_cast<int64_t>(t.w) * NT; z < padded; ++z) {  // alignment tail
                cja[t.ebase + z] = t.r0;
                cal[t.ebase + z] = 0.0;
                if (!a.value_symmetric) cau[t.ebase + z] = 0.0;
            }
            for (int32_t l = 0; l < NT; ++l) {
                const int64_t r = static_cast<int64_t>(t.r0) + l;
                const int32_t i = r < t.r1 ? rid[r] : -1;
                const int32_t len = i >= 0 ? a.ia[i + 1] - a.ia[i] : 0;
                for (int32_t q = 0; q < t.w; ++q) {
                    const int64_t e = t.ebase + static_cast<int64_t>(q) * NT + l;
                    if (q < len) {
                        const int64_t s = a.ia[i] + q;
                        cja[e] = pos[a.ja[s]];
                        cal[e] = a.al[s];
                        if (!a.value_symmetric) cau[e] = a.au[s];
                    } else {  // padding: own row, zero values (never gathered nor scattered)
                        cja[e] = static_cast<int32_t>(r);
                        cal[e] = 0.0;
                        if (!a.value_symmetric) cau[e] = 0.0;
                    }
                }
            }
        }
    }, 64);
    }
    // dispatch along diagonals b + D e (D > R): class e trails class e-1 by D blocks, so
    // (e, b)'s dependencies (e-1, b-R .. b+R) lie D - R diagonals earlier; all classes
    // are in flight at once over a window of ~D (C + 2) blocks (x, y L2-resident).
    // D B must cover the bandwidth plus the rows whose read-add-write phase is in flight:
    // every resident thread's row for the direct form (D = 4 R at C5: 1.72 ms vs 2.12 at
    // 2 R, profiles/r02_colored_wave_sweep.txt), only the consumer rows of the ring form.
    const void* fn = ring ? colored_ring_fn<T>(P) : colored_wave_fn<T>(P);
    const int smem = ring ? P.cr_stages * P.cr_stage_bytes : 0;
    if (ring) set_smem_limit(fn, smem);
    int occ = 0;
    CUDA_OK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, ring ? colored_ring_threads(P) : P.cw_nt, smem));
    const int per_sm = env_int("CSRC_GPU_CW_CTAS", std::max(occ, 1));
    const int grid_max = num_sms(P.device) * std::min(per_sm, std::max(occ, 1));
    int d_default = 4 * R;
    if (ring) {
        // class distance = bandwidth + slack x the consumer rows: a CTA holds ~5 claimed,
        // unfinished tickets, and 4x is the C5 optimum (more spills the window out of L2:
        // profiles/r02_colored_ring_sweeps.txt); when x and y fit L2 whole there is nothing
        // to spill and a wider distance only removes dependency waits (16x: C3 0.47 vs 0.56 ms,
        // C4 0.76 vs 0.88; profiles/r02c_colored_c2_c3_c4_defaults.txt); fp32 halves the window bytes
        const bool fits_l2 = 2.0 * static_cast<double>(npad) * sizeof(T) <= 96e6;
        const double slack = env_int("CSRC_GPU_CR_SLACK_PCT", fits_l2 ? 1600 : (sizeof(T) == 4 ? 600 : 400)) / 100.0;
        d_default = static_cast<int>(std::ceil((static_cast<double>(bw) + slack * grid_max * P.cw_nt) / static_cast<double>(B)));
    }
    const int D = std::max(R + 1, env_int("CSRC_GPU_CW_D", d_default));
    std::vector<int> order(P.cw_tasks);
    std::iota(order.begin(), order.end(), 0);
    auto key = [&](int t) {
        const int e = t / NB, b = t % NB;
        return std::make_tuple(b + D * e, e, b);
    };
    std::sort(order.begin(), order.end(), [&](int x, int y) { return key(x) < key(y); });
    std::vector<dev::CwTicket> tk;
    for (int t : order)
        for (const dev::CwTicket& c : chunks[t]) tk.push_back(c);
    P.cw_tickets = static_cast<int>(tk.size());
    upload(P.rid, rid.data(), rid.size());
    if (ring) {
        upload(P.cpk, cpk.data(), static_cast<size_t>(ne) + 16);
    } else {
        const size_t ne_up = static_cast<size_t>(std::max<int64_t>(ne, 4));
        upload(P.cja, cja.data(), ne_up);
        upload_values<T>(P.cal, cal.data(), ne_up);
        if (!a.value_symmetric) upload_values<T>(P.cau, cau.data(), ne_up);
    }
    upload_values<T>(P.cad, cad.data(), static_cast<size_t>(npad));
    upload(P.cw_tk, tk.data(), tk.size());
    upload(P.cw_nch, nch.data(), nch.size());
    P.cw_ctr.alloc(static_cast<size_t>(P.cw_tasks + 1) * 4);
    P.cw_xp.alloc(static_cast<size_t>(npad) * sizeof(T));
    P.cw_yp.alloc(static_cast<size_t>(npad) * sizeof(T));
    P.cw_grid = std::max(1, std::min(P.cw_tickets, grid_max));
    P.cw = true;
}

template <class T>
void setup_colored(Plan& P, const MatView& a, const std::vector<int32_t>& color, int n_colors) {
    P.n_colors = n_colors;
    if (env_int("CSRC_GPU_COLOR_WAVE", 1) != 0) {
        setup_colored_wave<T>(P, a, color, n_colors);
        return;
    }
    const index_t n = a.n;
    P.class_ptr.assign(n_colors + 1, 0);
    for (index_t i = 0; i < n; ++i) ++P.class_ptr[color[i] + 1];
    for (int c = 0; c < n_colors; ++c) P.class_ptr[c + 1] += P.class_ptr[c];
    std::vector<int32_t> rows(n);
    {
        std::vector<count_t> next(P.class_ptr.begin(), P.class_ptr.end() - 1);
        for (index_t i = 0; i < n; ++i) rows[next[color[i]]++] = i;  // ascending per class
    }
    std::vector<int64_t> cia(static_cast<size_t>(n) + 1, 0);
    for (index_t r = 0; r < n; ++r) cia[r + 1] = cia[r] + (a.ia[rows[r] + 1] - a.ia[rows[r]]);
    std::vector<int32_t> cja(static_cast<size_t>(a.k));
    std::vector<double> cal(static_cast<size_t>(a.k)), cau, cad(n);
    if (!a.value_symmetric) cau.resize(static_cast<size_t>(a.k));
    for (index_t r = 0; r < n; ++r) {
        const index_t i = rows[r];
        cad[r] = a.ad[i];
        count_t q = cia[r];
        for (index_t t = a.ia[i]; t < a.ia[i + 1]; ++t, ++q) {
            cja[q] = a.ja[t];
            cal[q] = a.al[t];
            if (!a.value_symmetric) cau[q] = a.au[t];
        }
    }
    upload(P.rid, rows.data(), rows.size());
    upload(P.cia, cia.data(), cia.size());
    upload(P.cja, cja.data(), cja.size());
    upload_values<T>(P.cal, cal.data(), cal.size());
    if (!a.value_symmetric) upload_values<T>(P.cau, cau.data(), cau.size());
    upload_values<T>(P.cad, cad.data(), cad.size());
}

int pick_lanes(count_t k, index_t n) {
    const double avg = n ? static_cast<double>(k) / n : 1.0;
    if (avg <= 2.5) return 2;
    if (avg <= 5) return 4;
    if (avg <= 10) return 8;
    if (avg <= 20) return 16;
    return 32;
}

int grid_for(int device, int64_t work, int per_block);

// -------------------------------------------------------------- gather
// Entry stream per row q: lower pairs of q (ja / al, CSRC order), then the
// pairs (r, q), r > q ascending, with their au (normal product) or al
// (transpose) value. eval_t only exists for value-unsymmetric matrices.
// Dictionary of per-row column-offset patterns (offsets c - q in entry
// order); pbase[q] = start of row q's pattern in pat_off. Gives up (returns
// false) past 65535 patterns or 1 M stored offsets: then the plan keeps
// explicit column indices.
// One dictionary of row offset patterns (local to a slice of rows, or global).
struct PatternDict {
    std::vector<int32_t> off, ptr{0};
    std::unordered_map<uint64_t, std::vector<int32_t>> by_hash;
    // id of the pattern (o[0..len)), inserting it if new; -1 past the limits
    int32_t find_or_add(const int32_t* o, int32_t len, uint64_t h) {
        auto& cand = by_hash[h];
        for (int32_t p : cand) {
            const int32_t p0 = ptr[p];
            if (ptr[p + 1] - p0 != len) continue;
            if (std::equal(o, o + len, off.begin() + p0)) return p;
        }
        const int32_t id = static_cast<int32_t>(ptr.size()) - 1;
        if (id >= 65535 || off.size() + len > (size_t(1) << 20)) return -1;
        off.insert(off.end(), o, o + len);
        ptr.push_back(static_cast<int32_t>(off.size()));
        cand.push_back(id);
        return id;
    }
};

inline uint64_t pattern_hash(const int32_t* o, int32_t len) {
    uint64_t h = 0x9E3779B97F4A7C15ull ^ static_cast<uint64_t>(len);
    for (int32_t j = 0; j < len; ++j) h = (h ^ static_cast<uint32_t>(o[j])) * 0x100000001B3ull;
    return h;
}

// Dictionary of per-row column-offset patterns (offsets c - q in entry
// order); pbase[q] = start of row q's pattern in pat_off. Gives up (returns
// false) past 65535 patterns or 1 M stored offsets: then the plan keeps
// explicit column indices. Row slices build local dictionaries in parallel;
// merging them in slice order reproduces the serial first-occurrence order,
// so the table and pbase are the same whatever the thread count.
bool find_row_patterns(index_t n, const std::vector<int32_t>& eptr, const HVec<int32_t>& eidx,
                       std::vector<int32_t>& pbase, std::vector<int32_t>& pat_off, int32_t* n_patterns) {
    pbase.assign(static_cast<size_t>(n), 0);
    std::vector<int32_t> lid(static_cast<size_t>(n));
    std::vector<PatternDict> local(64);
    std::vector<char> failed(64, 0);
    int slices = 0;
    parallel_slices(n, [&](int t, int64_t b, int64_t e) {
        PatternDict& D = local[t];
        std::vector<int32_t> o;
        int32_t prev = -1;  // consecutive rows usually share a pattern: try it first
        for (index_t q = static_cast<index_t>(b); q < e; ++q) {
            const int32_t e0 = eptr[q], len = eptr[q + 1] - e0;
            o.resize(static_cast<size_t>(len));
            for (int32_t j = 0; j < len; ++j) o[j] = eidx[e0 + j] - q;
            if (prev >= 0 && D.ptr[prev + 1] - D.ptr[prev] == len &&
                std::equal(o.begin(), o.end(), D.off.begin() + D.ptr[prev])) {
                lid[q] = prev;
                continue;
            }
            const int32_t id = D.find_or_add(o.data(), len, pattern_hash(o.data(), len));
            if (id < 0) {
                failed[t] = 1;
                return;
            }
            lid[q] = prev = id;
        }
    });
    for (int t = 0; t < 64; ++t) {
        if (failed[t]) return false;
        if (local[t].ptr.size() > 1 || t == 0) slices = t + 1;
    }
    // merge in slice order: global ids by first occurrence, as a serial pass
    PatternDict G;
    std::vector<std::vector<int32_t>> to_global(static_cast<size_t>(slices));
    for (int t = 0; t < slices; ++t) {
        const PatternDict& D = local[t];
        const int np = static_cast<int>(D.ptr.size()) - 1;
        to_global[t].resize(static_cast<size_t>(np));
        for (int p = 0; p < np; ++p) {
            const int32_t* o = D.off.data() + D.ptr[p];
            const int32_t len = D.ptr[p + 1] - D.ptr[p];
            const int32_t g = G.find_or_add(o, len, pattern_hash(o, len));
            if (g < 0) return false;
            to_global[t][p] = G.ptr[g];  // pattern start in the global table
        }
    }
    parallel_slices(n, [&](int t, int64_t b, int64_t e) {
        for (index_t q = static_cast<index_t>(b); q < e; ++q) pbase[q] = to_global[t][lid[q]];
    });
    *n_patterns = static_cast<int32_t>(G.ptr.size()) - 1;
    pat_off = std::move(G.off);
    if (pat_off.empty()) pat_off.push_back(0);  // keep the device table non-empty
    return true;
}

// row-setup area per staging buffer (0 = the kernel loads eptr / pbase from global memory)
int gather_rs_bytes(const Plan& P) {
    if (!P.gather_rs || P.gather_xs) return 0;
    return dev::gather_rows_bytes(P.gather_nt / P.gather_lanes) * (P.gather_pat ? 2 : 1);
}

template <class T>
int gather_stage_smem(const Plan& P) {
    return 16 + P.gather_nb * ((P.gather_pat ? 0 : dev::gather_idx_bytes(P.gather_cap)) +
                               dev::gather_val_bytes<T>(P.gather_cap) + (P.gather_xs ? P.xs_bytes : 0) +
                               gather_rs_bytes(P));
}

// pattern form of the staged kernel: 0 explicit columns, 1 row patterns, 2 patterns + staged x
int gather_pf(const Plan& P) { return P.gather_pat ? (P.gather_xs ? 2 : 1) : 0; }

template <class T, int L, int U, int NB, int MINB>
void* gather_stage_fn_M(int pf) {
    switch (pf) {
        case 2: return reinterpret_cast<void*>(&dev::k_gather_staged<T, L, U, NB, 2, MINB>);
        case 1: return reinterpret_cast<void*>(&dev::k_gather_staged<T, L, U, NB, 1, MINB>);
        default: return reinterpret_cast<void*>(&dev::k_gather_staged<T, L, U, NB, 0, MINB>);
    }
}

template <class T, int L, int U, int NB>
void* gather_stage_fn_NB(int pf, int minb) {
    switch (minb) {
        case 8: return gather_stage_fn_M<T, L, U, NB, 8>(pf);
        case 6: return gather_stage_fn_M<T, L, U, NB, 6>(pf);
        case 5: return gather_stage_fn_M<T, L, U, NB, 5>(pf);
        default: return gather_stage_fn_M<T, L, U, NB, 1>(pf);
    }
}

template <class T, int L>
void* gather_stage_fn_L(int U, int NB, int pf, int minb) {
    if (U == 8)
        return NB == 2 ? gather_stage_fn_NB<T, L, 8, 2>(pf, minb) : gather_stage_fn_NB<T, L, 8, 1>(pf, minb);
    return NB == 2 ? gather_stage_fn_NB<T, L, 4, 2>(pf, minb) : gather_stage_fn_NB<T, L, 4, 1>(pf, minb);
}

template <class T>
void* gather_stage_fn(const Plan& P) {
    const int pf = gather_pf(P);
    switch (P.gather_lanes) {
        case 1:  // one row per thread: U = 8, one buffer, no staged x (setup_gather); opt-in 6-block bound
            if (pf == 1 && P.gather_minb == 6) return reinterpret_cast<void*>(&dev::k_gather_staged<T, 1, 8, 1, 1, 6>);
            return pf == 1 ? reinterpret_cast<void*>(&dev::k_gather_staged<T, 1, 8, 1, 1, 1>)
                           : reinterpret_cast<void*>(&dev::k_gather_staged<T, 1, 8, 1, 0, 1>);
        case 2: return gather_stage_fn_L<T, 2>(P.gather_u, P.gather_nb, pf, P.gather_minb);
        case 8: return gather_stage_fn_L<T, 8>(P.gather_u, P.gather_nb, pf, P.gather_minb);
        default: return gather_stage_fn_L<T, 4>(P.gather_u, P.gather_nb, pf, P.gather_minb);
    }
}

// Staged-x form (k_gather_staged, PF = 2): the pattern dictionary's column
// offsets grouped into clusters (a new cluster after a gap of more than 32);
// row block [q0, q0 + R) reads x only on [q0 + clo_k, q0 + R + chi_k), copied
// by TMA next to the values. Per alignment phase ph of the x pointer
// (16-byte grain), xs_tab[ph][i] = cbase_k + ((ph + clo_k) mod m) + (d_i - clo_k)
// locates pattern entry i's x value relative to the row's local index.
// Returns false (staged x off) past 32 clusters or 24 KB of x per row block.
template <class T>
bool setup_staged_x(Plan& P, const std::vector<int32_t>& pat_off) {
    const int R = P.gather_nt / P.gather_lanes;
    const int m = 16 / static_cast<int>(sizeof(T));
    std::vector<int32_t> offs(pat_off.begin(), pat_off.end());
    std::sort(offs.begin(), offs.end());
    offs.erase(std::unique(offs.begin(), offs.end()), offs.end());
    if (offs.empty()) return false;
    std::vector<int32_t> clo, chi, cbase;
    for (size_t i = 0; i < offs.size(); ++i) {
        if (clo.empty() || static_cast<int64_t>(offs[i]) - chi.back() > 32) {
            clo.push_back(offs[i]);
            chi.push_back(offs[i]);
        } else {
            chi.back() = offs[i];
        }
    }
    if (clo.size() > 32) return false;
    int64_t acc = 0;
    for (size_t k = 0; k < clo.size(); ++k) {
        cbase.push_back(static_cast<int32_t>(acc));
        const int64_t cap = R + (static_cast<int64_t>(chi[k]) - clo[k]) + 2 * m;
        acc += (cap + m - 1) / m * m;
    }
    const int64_t bytes = acc * static_cast<int64_t>(sizeof(T));
    if (bytes > 24 * 1024) return false;
    const size_t tl = pat_off.size();
    std::vector<int32_t> tab(tl * m);
    for (int ph = 0; ph < m; ++ph)
        for (size_t i = 0; i < tl; ++i) {
            const int32_t d = pat_off[i];
            const size_t k = static_cast<size_t>(std::upper_bound(clo.begin(), clo.end(), d) - clo.begin()) - 1;
            const int32_t pad = static_cast<int32_t>(((ph + static_cast<int64_t>(clo[k])) % m + m) % m);
            tab[ph * tl + i] = cbase[k] + pad + (d - clo[k]);
        }
    upload(P.xs_tab, tab.data(), tab.size());
    upload(P.xs_clo, clo.data(), clo.size());
    upload(P.xs_chi, chi.data(), chi.size());
    upload(P.xs_cbase, cbase.data(), cbase.size());
    P.xs_clusters = static_cast<int>(clo.size());
    P.xs_tab_len = static_cast<int>(tl);
    P.xs_bytes = static_cast<int>((bytes + 15) / 16 * 16);
    return true;
}

template <class T, int L, bool PAT>
void* sell_fn_LP(int u) {
    switch (u) {
        case 4: return reinterpret_cast<void*>(&dev::k_gather_sell<T, L, PAT, 4>);
        case 9: return reinterpret_cast<void*>(&dev::k_gather_sell<T, L, PAT, 9>);
        case 12: return reinterpret_cast<void*>(&dev::k_gather_sell<T, L, PAT, 12>);
        case 14: return reinterpret_cast<void*>(&dev::k_gather_sell<T, L, PAT, 14>);
        default: return reinterpret_cast<void*>(&dev::k_gather_sell<T, L, PAT, 8>);
    }
}

template <class T>
void* sell_fn(const Plan& P) {
    const bool pat = P.gather_pat != 0;
    switch (P.sell_lanes) {
        case 2: return pat ? sell_fn_LP<T, 2, true>(P.sell_u) : sell_fn_LP<T, 2, false>(P.sell_u);
        case 4: return pat ? sell_fn_LP<T, 4, true>(P.sell_u) : sell_fn_LP<T, 4, false>(P.sell_u);
        default: return pat ? sell_fn_LP<T, 1, true>(P.sell_u) : sell_fn_LP<T, 1, false>(P.sell_u);
    }
}

// Sliced layout of the entry stream (gather.cuh k_gather_sell): slice s =
// rows [H s, H s + H), H = 32 / L; width = ceil(longest row / L) steps of 32
// slots; entry j of local row rl at sbase[s] + 32 (j / L) + L rl + j % L;
// padding slots hold zeros and are never read.
template <class T>
void setup_sell(Plan& P, index_t n, const std::vector<int32_t>& eptr, const HVec<int32_t>& eidx,
                const HVec<double>& ev, const HVec<double>& evt, bool value_symmetric,
                const std::vector<int32_t>& pbase, const std::vector<int32_t>& pat_off) {
    const double avg = n ? static_cast<double>(eptr[n]) / n : 0.0;
    // lanes per row: rows of <= 40 entries (27-point stencils) split over 2
    // lanes, longer rows (81-entry elasticity) one lane (profiles/r01_sweep_sell*.txt)
    const int L = env_int("CSRC_GPU_SELL_L", 1);  // 2 / 4 lanes lost on every config (r01_sweep_sell2.txt)
    P.sell_lanes = (L == 2 || L == 4) ? L : 1;
    const int H = 32 / P.sell_lanes;
    const int64_t ns = (static_cast<int64_t>(n) + H - 1) / H;
    std::vector<int32_t> sbase(static_cast<size_t>(ns) + 1, 0);
    int32_t maxlen = 0;
    for (int64_t sl = 0; sl < ns; ++sl) {
        int32_t w = 0;
        for (int64_t r = sl * H; r < std::min<int64_t>(n, sl * H + H); ++r) w = std::max(w, eptr[r + 1] - eptr[r]);
        maxlen = std::max(maxlen, w);
        const int64_t steps = (w + P.sell_lanes - 1) / P.sell_lanes;
        const int64_t next = static_cast<int64_t>(sbase[sl]) + 32 * steps;
        if (next > INT32_MAX) throw Error("gather plan: padded slice layout exceeds 2^31 entries");
        sbase[sl + 1] = static_cast<int32_t>(next);
    }
    // pattern form: offset table in shared memory (<= 16 K entries), rows < 2^11 entries
    const bool pat = P.gather_pat && maxlen < 2048 && pat_off.size() <= (size_t(1) << 14);
    P.gather_pat = pat ? 1 : 0;
    const size_t tot = static_cast<size_t>(sbase[ns]);
    P.sell_entries = static_cast<int64_t>(tot);
    std::vector<int32_t> rmeta(static_cast<size_t>(n));
    // padding slots are never read: no value-initialisation (parallel first touch)
    HVec<int32_t> sidx(pat ? 0 : tot);
    HVec<double> sv(tot), svt(value_symmetric ? 0 : tot);
    const int Ln = P.sell_lanes;
    parallel_slices(ns, [&](int, int64_t s0, int64_t s1) {
        for (int64_t sl = s0; sl < s1; ++sl)
            for (int64_t r = sl * H; r < std::min<int64_t>(n, sl * H + H); ++r) {
                const int32_t len = eptr[r + 1] - eptr[r];
                rmeta[r] = pat ? (pbase[r] | (len << 20)) : len;
                const size_t b = static_cast<size_t>(sbase[sl]) + static_cast<size_t>(Ln * (r - sl * H));
                for (int32_t j = 0; j < len; ++j) {
                    const size_t d = b + 32 * static_cast<size_t>(j / Ln) + static_cast<size_t>(j % Ln);
                    sv[d] = ev[eptr[r] + j];
                    if (!value_symmetric) svt[d] = evt[eptr[r] + j];
                    if (!pat) sidx[d] = eidx[eptr[r] + j];
                }
            }
    }, 1024);
    upload(P.sbase, sbase.data(), sbase.size());
    upload(P.rmeta, rmeta.data(), rmeta.size());
    upload_values<T>(P.sval, sv.data(), sv.size());
    if (!value_symmetric) upload_values<T>(P.sval_t, svt.data(), svt.size());
    if (pat) upload(P.pat_off, pat_off.data(), pat_off.size());
    else upload(P.sidx, sidx.data(), sidx.size());
    if (!pat) P.n_patterns = 0;
    const int u = env_int("CSRC_GPU_SELL_U", 8);
    P.sell_u = (u == 4 || u == 9 || u == 12 || u == 14) ? u : 8;
    P.gather_sell = 1;
    P.gather_buf = 0;
    P.sell_pat_len = pat ? static_cast<int>(pat_off.size()) : 0;
    void* fn = sell_fn<T>(P);
    const int smem = 4 * P.sell_pat_len;
    set_smem_limit(reinterpret_cast<const void*>(fn), smem);
    int occ = 0;
    CUDA_OK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, 256, smem));
    const int64_t blocks = (ns + 7) / 8;
    P.sell_grid = static_cast<int>(std::max<int64_t>(
        1, std::min<int64_t>(blocks, static_cast<int64_t>(num_sms(P.device)) * std::max(occ, 1))));
}

template <class T>
void finish_gather(Plan& P, index_t n, bool band, std::vector<int32_t>& eptr, HVec<int32_t>& eidx,
                   HVec<double>& ev, HVec<double>& evt, bool value_symmetric, bool trace,
                   DevEntries* dv = nullptr);

// Whole-matrix gather entries on the device: pairs stably radix-sorted by
// column give each target row its upper pairs in ascending source row, the
// serial host builder's order, so both builders produce the same plan.
// Returns eptr and eidx on the host (patterns, pipeline chunks); the values
// stay on the device.
void build_entries_device(Plan& P, const MatView& a, std::vector<int32_t>& eptr, HVec<int32_t>& eidx,
                          DevEntries& D) {
    const index_t n = a.n;
    const int64_t k = a.k, ne = 2 * k;
    cudaStream_t st = P.stream;
    DevBuf ia, ja, al, au, erow, up, cnt, ep, key, val, key2, val2, ust;
    upload(ia, a.ia, static_cast<size_t>(n) + 1);
    upload(ja, a.ja, static_cast<size_t>(k));
    upload(al, a.al, static_cast<size_t>(k));
    if (!a.value_symmetric) upload(au, a.au, static_cast<size_t>(k));
    erow.alloc(static_cast<size_t>(k) * 4);
    up.alloc((static_cast<size_t>(n) + 1) * 4);
    cnt.alloc((static_cast<size_t>(n) + 1) * 4);
    ep.alloc((static_cast<size_t>(n) + 1) * 4);
    const unsigned gb = static_cast<unsigned>(std::min<int64_t>(std::max<int64_t>(1, (k + 255) / 256), 1 << 20));
    const unsigned gn = static_cast<unsigned>(std::min<int64_t>(std::max<int64_t>(1, (n + 255) / 256), 1 << 20));
    CUDA_OK(cudaMemsetAsync(up.p, 0, (static_cast<size_t>(n) + 1) * 4, st));
    CUDA_OK(cudaMemsetAsync(cnt.p, 0, (static_cast<size_t>(n) + 1) * 4, st));
    dev::k_pair_rows<<<gn, 256, 0, st>>>(n, ia.as<int32_t>(), erow.as<int32_t>());
    dev::k_upper_counts<<<gb, 256, 0, st>>>(k, ja.as<int32_t>(), up.as<int32_t>());
    dev::k_row_counts<<<gn, 256, 0, st>>>(n, ia.as<int32_t>(), up.as<int32_t>(), cnt.as<int32_t>());
    CUDA_OK(cudaGetLastError());
    size_t tmp_bytes = 0;
    CUDA_OK(cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, cnt.as<int32_t>(), ep.as<int32_t>(), n + 1, st));
    {
        DevBuf tmp;
        tmp.alloc(tmp_bytes);
        CUDA_OK(cub::DeviceScan::ExclusiveSum(tmp.p, tmp_bytes, cnt.as<int32_t>(), ep.as<int32_t>(), n + 1, st));
        CUDA_OK(cudaStreamSynchronize(st));
    }
    D.eidx.alloc(static_cast<size_t>(ne) * 4);
    D.ev.alloc(static_cast<size_t>(ne) * 8);
    if (!a.value_symmetric) D.evt.alloc(static_cast<size_t>(ne) * 8);
    const double* aup = a.value_symmetric ? nullptr : au.as<double>();
    dev::k_place_lower<<<gb, 256, 0, st>>>(k, erow.as<int32_t>(), ia.as<int32_t>(), ja.as<int32_t>(),
                                           al.as<double>(), aup, ep.as<int32_t>(), D.eidx.as<int32_t>(),
                                           D.ev.as<double>(), D.evt.as<double>());
    CUDA_OK(cudaGetLastError());
    // stable LSD radix sort of (column, pair) -> pairs grouped by column, rows ascending
    key.alloc(static_cast<size_t>(k) * 4);
    val.alloc(static_cast<size_t>(k) * 4);
    key2.alloc(static_cast<size_t>(k) * 4);
    val2.alloc(static_cast<size_t>(k) * 4);
    CUDA_OK(cudaMemcpyAsync(key.p, ja.p, static_cast<size_t>(k) * 4, cudaMemcpyDeviceToDevice, st));
    dev::k_iota<<<gb, 256, 0, st>>>(k, val.as<int32_t>());  // pair ids 0..k-1
    CUDA_OK(cudaGetLastError());
    int bits = 1;
    while ((int64_t{1} << bits) < n) ++bits;
    cub::DoubleBuffer<int32_t> kb(key.as<int32_t>(), key2.as<int32_t>()), vb(val.as<int32_t>(), val2.as<int32_t>());
    tmp_bytes = 0;
    CUDA_OK(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, kb, vb, static_cast<int>(k), 0, bits, st));
    {
        DevBuf tmp;
        tmp.alloc(tmp_bytes);
        CUDA_OK(cub::DeviceRadixSort::SortPairs(tmp.p, tmp_bytes, kb, vb, static_cast<int>(k), 0, bits, st));
        ust.alloc((static_cast<size_t>(n) + 1) * 4);
        size_t tb2 = 0;
        CUDA_OK(cub::DeviceScan::ExclusiveSum(nullptr, tb2, up.as<int32_t>(), ust.as<int32_t>(), n + 1, st));
        DevBuf tmp2;
        tmp2.alloc(tb2);
        CUDA_OK(cub::DeviceScan::ExclusiveSum(tmp2.p, tb2, up.as<int32_t>(), ust.as<int32_t>(), n + 1, st));
        dev::k_place_upper<<<gb, 256, 0, st>>>(k, kb.Current(), vb.Current(), ust.as<int32_t>(), ia.as<int32_t>(),
                                               erow.as<int32_t>(), al.as<double>(), aup, ep.as<int32_t>(),
                                               D.eidx.as<int32_t>(), D.ev.as<double>(), D.evt.as<double>());
        CUDA_OK(cudaGetLastError());
        CUDA_OK(cudaStreamSynchronize(st));
    }
    eptr.resize(static_cast<size_t>(n) + 1);
    CUDA_OK(cudaMemcpy(eptr.data(), ep.p, (static_cast<size_t>(n) + 1) * 4, cudaMemcpyDeviceToHost));
    eidx.resize(static_cast<size_t>(ne));
    {
        HostLink hl(st);
        hl.d2h(eidx.data(), D.eidx.p, static_cast<size_t>(ne) * 4);
    }
}

template <class T>
void setup_gather(Plan& P, const MatView& a) {
    // rows [r0, r1) of the global matrix (the whole matrix unless a band plan);
    // entry columns are stored in band-row coordinates (c - r0, negative below
    // the band) and the kernels read x through a pointer shifted by r0 - lo, so
    // the device x holds [lo, x_hi) and y holds the band rows only.
    const index_t N = a.n;
    const index_t r0 = P.row_begin, r1 = P.row_end;
    const index_t n = r1 - r0;
    const bool band = n != N;
    if (2 * static_cast<int64_t>(a.k) > INT32_MAX)
        throw Error("gather plan: more than 2^31 off-diagonal entries (use the windowed kernel)");
    // CSRC_GPU_PLAN_TRACE=1: phase times of the plan build on stderr (diagnostics)
    const bool trace = env_int("CSRC_GPU_PLAN_TRACE", 0) != 0;
    if (!band && a.k >= (int64_t{1} << 20) && env_int("CSRC_GPU_PLAN_DEVICE", 0) != 0) {
        // opt-in (CSRC_GPU_PLAN_DEVICE=1): the transposition on the device. The same
        // plan bit for bit, but not faster: moving the 4.8 GB of CSRC arrays up and
        // the 1.7 GB of entry columns down costs what the host transposition does
        // (C5 1.29 s vs 1.15 s; profiles/r01_plan_build_trace_device.txt)
        const auto t0 = std::chrono::steady_clock::now();
        std::vector<int32_t> eptr;
        HVec<int32_t> eidx;
        HVec<double> ev, evt;
        DevEntries D;
        build_entries_device(P, a, eptr, eidx, D);
        P.x_hi = r1;
        P.gi0 = 0;
        P.gi1 = n;  // whole matrix: every column is one of the plan's rows
        if (trace)
            std::fprintf(stderr, "gather plan: %-22s %8.1f ms\n", "device entries",
                         std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
        finish_gather<T>(P, n, band, eptr, eidx, ev, evt, a.value_symmetric, trace, &D);
        return;
    }
    auto t_last = std::chrono::steady_clock::now();
    auto mark = [&](const char* what) {
        if (!trace) return;
        const auto t = std::chrono::steady_clock::now();
        std::fprintf(stderr, "gather plan: %-22s %8.1f ms\n", what,
                     std::chrono::duration<double, std::milli>(t - t_last).count());
        t_last = t;
    };
    // upper entries of q = the pairs (r, q), r > q: count them per column
    // (relaxed atomic increments) and find x_hi, over row slices in parallel
    std::vector<int32_t> up(static_cast<size_t>(n) + 1, 0);
    std::vector<index_t> xhi_t(64, r1);
    parallel_slices(N - (r0 + 1), [&](int t, int64_t b, int64_t e) {
        index_t xh = r1;
        for (index_t r = static_cast<index_t>(r0 + 1 + b); r < r0 + 1 + e; ++r)
            for (index_t q = a.ia[r]; q < a.ia[r + 1]; ++q)
                if (a.ja[q] >= r0 && a.ja[q] < r1) {
                    __atomic_fetch_add(&up[a.ja[q] - r0 + 1], 1, __ATOMIC_RELAXED);
                    xh = std::max(xh, r + 1);
                }
        xhi_t[t] = xh;
    });
    index_t x_hi = r1;
    for (index_t v : xhi_t) x_hi = std::max(x_hi, v);
    P.x_hi = x_hi;
    mark("upper counts");
    std::vector<int32_t> eptr(static_cast<size_t>(n) + 1, 0);
    for (index_t q = 0; q < n; ++q)
        eptr[q + 1] = eptr[q] + (a.ia[r0 + q + 1] - a.ia[r0 + q]) + up[q + 1];
    const size_t ne = static_cast<size_t>(eptr[n]);
    // no value-initialisation: every slot is written below, and the first-touch
    // page faults of these multi-GB arrays happen in the parallel fill
    HVec<int32_t> eidx(ne);
    HVec<double> ev(ne), evt(a.value_symmetric ? 0 : ne);
    std::vector<int32_t> next(static_cast<size_t>(n));
    parallel_slices(n, [&](int, int64_t b, int64_t e) {  // lower pairs, row by row
        for (index_t q = static_cast<index_t>(b); q < e; ++q) {
            int32_t w = eptr[q];
            for (index_t t = a.ia[r0 + q]; t < a.ia[r0 + q + 1]; ++t, ++w) {
                eidx[w] = a.ja[t] - r0;
                ev[w] = a.al[t];
                if (!a.value_symmetric) evt[w] = a.au[t];
            }
            next[q] = w;  // upper entries of q start here
        }
    });
    mark("alloc + lower pairs");
    // upper pairs: thread t owns the target rows (columns) [qb, qe) and walks the
    // rows r > qb in ascending order, so each target's upper entries land
    // sorted by r -- the same order as a serial pass, whatever the thread count.
    // Rows whose smallest column (ja ascends within a row) is >= the slice end
    // cannot name one of its targets.
    parallel_slices(n, [&](int, int64_t qb, int64_t qe) {
        const index_t lo_col = static_cast<index_t>(r0 + qb), hi_col = static_cast<index_t>(r0 + qe);
        int64_t remaining = 0;  // upper entries of the slice still to place: stop at 0
        for (int64_t q = qb; q < qe; ++q) remaining += up[q + 1];
        for (index_t r = std::max<index_t>(r0 + 1, lo_col + 1); r < N && remaining > 0; ++r) {
            const index_t t0 = a.ia[r], t1 = a.ia[r + 1];
            if (t0 == t1 || a.ja[t0] >= hi_col) continue;
            for (index_t t = t0; t < t1; ++t) {
                const index_t c = a.ja[t];
                if (c < lo_col) continue;
                if (c >= hi_col) break;
                const int32_t w = next[c - r0]++;
                eidx[w] = r - r0;
                ev[w] = a.value_symmetric ? a.al[t] : a.au[t];
                if (!a.value_symmetric) evt[w] = a.al[t];
                --remaining;
            }
        }
    });
    mark("upper pairs");
    {
        // interior rows of a band: all columns inside the band's own rows [0, n)
        std::vector<index_t> b0_t(64, 0), b1_t(64, n);
        parallel_slices(n, [&](int t, int64_t qb, int64_t qe) {
            index_t lo = 0, hi = n;
            for (index_t q = static_cast<index_t>(qb); q < qe; ++q)
                for (int32_t e = eptr[q]; e < eptr[q + 1]; ++e) {
                    if (eidx[e] < 0) lo = std::max(lo, q + 1);
                    if (eidx[e] >= n) hi = std::min(hi, q);
                }
            b0_t[t] = lo;
            b1_t[t] = hi;
        });
        index_t b0 = 0, b1 = n;
        for (int t = 0; t < 64; ++t) {
            b0 = std::max(b0, b0_t[t]);
            b1 = std::min(b1, b1_t[t]);
        }
        const index_t a0 = (b0 + 255) / 256 * 256, a1 = b1 == n ? n : b1 / 256 * 256;
        P.gi0 = std::min(a0, n);
        P.gi1 = std::max(P.gi0, a1);
    }
    mark("interior split");
    finish_gather<T>(P, n, band, eptr, eidx, ev, evt, a.value_symmetric, trace);
}

// Second half of a gather plan, shared by the CSRC plans (setup_gather) and
// the CSR plans (setup_gather_csr): host pipeline chunks, row patterns, kernel
// form (staged / sliced / rows), uploads.
template <class T>
void finish_gather(Plan& P, index_t n, bool band, std::vector<int32_t>& eptr, HVec<int32_t>& eidx,
                   HVec<double>& ev, HVec<double>& evt, bool value_symmetric, bool trace, DevEntries* dv) {
    const size_t ne = static_cast<size_t>(eptr[n]);
    auto t_last = std::chrono::steady_clock::now();
    auto mark = [&](const char* what) {
        if (!trace) return;
        const auto t = std::chrono::steady_clock::now();
        std::fprintf(stderr, "gather plan: %-22s %8.1f ms\n", what,
                     std::chrono::duration<double, std::milli>(t - t_last).count());
        t_last = t;
    };
    const double avg = n ? static_cast<double>(ne) / n : 0.0;
    // lanes per row: stencil rows (<= 40 entries) 2 for fp64, 1 for fp32 (C5 fp32
    // 0.422 vs 0.470 ms; fp64 0.631 vs 0.747 ms with 1: profiles/r01_sweep_gather_one_lane.txt)
    {
        const int dflt = avg <= 40 ? (sizeof(T) == 4 ? 1 : 2) : avg <= 128 ? 4 : 8;
        const int l = env_int("CSRC_GPU_GLANES", dflt);
        // only the instantiated lane counts: R = nt / lanes must match the kernel's own
        P.gather_lanes = (l == 1 || l == 2 || l == 4 || l == 8 || l == 16) ? l : dflt;
    }
    P.gather_pf = env_int("CSRC_GPU_GPF", 0);
    P.gather_bpsm = env_int("CSRC_GPU_GBPSM", 16);  // 256-thread blocks per SM
    if (!band) {
        // host pipeline: row chunks on multiples of 256 rows (any lane count's block).
        // Ramped sizes (in 64ths of n): a small first chunk starts the y download
        // early, small last chunks shorten the compute + download tail after the
        // last x chunk lands. CSRC_GPU_HOST_CHUNKS=c forces c equal chunks.
        P.hchunk.clear();
        const int forced = env_int("CSRC_GPU_HOST_CHUNKS", 0);
        std::vector<int> units;
        if (const char* us = std::getenv("CSRC_GPU_HOST_UNITS")) {  // e.g. "1,2,4,8,8,4,2,1"
            for (const char* q = us; *q;) {
                const int u = std::atoi(q);
                if (u > 0) units.push_back(u);
                while (*q && *q != ',') ++q;
                if (*q == ',') ++q;
            }
        }
        if (!units.empty())
            ;
        else if (forced > 0)
            units.assign(forced, 1);
        else if (n >= (int64_t(1) << 20))
            units = {2, 4, 8, 8, 8, 8, 8, 8, 4, 2, 2, 1, 1};
        else
            units = {1};
        int64_t tot = 0;
        for (int u : units) tot += u;
        int64_t acc = 0;
        P.hchunk.push_back(0);
        for (int u : units) {
            acc += u;
            int64_t b = (n * acc / tot + 255) / 256 * 256;
            b = std::min<int64_t>(b, n);
            if (b > P.hchunk.back()) P.hchunk.push_back(static_cast<int32_t>(b));
        }
        if (P.hchunk.back() != n) P.hchunk.push_back(n);
        const int nc = static_cast<int>(P.hchunk.size()) - 1;
        P.hneed.assign(nc, 0);
        std::vector<int32_t> hi_col(nc);
        std::vector<std::thread> pool;
        for (int c = 0; c < nc; ++c)
            pool.emplace_back([&, c] {
                int32_t hi = P.hchunk[c + 1] - 1;  // the diagonal reads x[row]
                for (int64_t e = eptr[P.hchunk[c]]; e < eptr[P.hchunk[c + 1]]; ++e) hi = std::max(hi, eidx[e]);
                hi_col[c] = hi;
            });
        for (auto& th : pool) th.join();
        // x chunks: by default x chunk c ends at the highest column row chunk c
        // reads, so chunk c's product starts once x chunk c has landed (the
        // halo of the next rows comes with it) instead of waiting for all of
        // x chunk c + 1; CSRC_GPU_HOST_XHALO=0 keeps x chunks = row chunks.
        if (env_int("CSRC_GPU_HOST_XHALO", 1) != 0) {
            P.xchunk.assign(1, 0);
            for (int c = 0; c < nc; ++c) {
                const int32_t e = c + 1 == nc ? static_cast<int32_t>(n)
                                              : std::min<int32_t>(static_cast<int32_t>(n),
                                                                  std::max(P.hchunk[c + 1], hi_col[c] + 1));
                P.xchunk.push_back(std::max(P.xchunk.back(), e));
            }
        } else {
            P.xchunk = P.hchunk;
        }
        for (int c = 0; c < nc; ++c)  // x chunk holding column hi
            P.hneed[c] = static_cast<int32_t>(std::upper_bound(P.xchunk.begin(), P.xchunk.end() - 1, hi_col[c]) -
                                              P.xchunk.begin()) - 1;
    }
    // staged form (k_gather_staged): U x-gathers in flight per lane, NB buffers,
    // NT threads per block; the row-pattern form when the rows repeat a small
    // dictionary of column-offset patterns
    P.gather_u = env_int("CSRC_GPU_GU", avg / P.gather_lanes <= 16 ? 8 : 4) == 8 ? 8 : 4;
    P.gather_nb = env_int("CSRC_GPU_GNB", 1) == 2 ? 2 : 1;
    // row setup staged with the values lost 1.5-3.5 % (profiles/r01_sweep_gather_row_setup.txt): opt-in
    P.gather_rs = env_int("CSRC_GPU_GROWS", 0) != 0 ? 1 : 0;
    {
        // 128-thread blocks (64 rows) for fp64: C5 0.631 ms vs 0.689 ms at 256 and
        // 0.664 at 64; fp32 keeps 256 (0.466 vs 0.558 ms)
        // (profiles/r01_sweep_gather_block_threads{,_64}.txt)
        const int nt = env_int("CSRC_GPU_GNT", sizeof(T) == 8 ? 128 : 256);
        P.gather_nt = (nt == 64 || nt == 128) ? nt : 256;
    }
    const int minb_env = env_int("CSRC_GPU_GMINB", -1);  // read once; -1 = per-shape default
    P.gather_minb = (minb_env == 8 || minb_env == 6 || minb_env == 5) ? minb_env : 1;
    mark("host pipeline chunks");
    std::vector<int32_t> pbase, pat_off;
    const bool has_pat = P.gather_lanes <= 8 && find_row_patterns(n, eptr, eidx, pbase, pat_off, &P.n_patterns);
    mark("row patterns");
    P.gather_pat = has_pat && env_int("CSRC_GPU_GPATTERN", 1) != 0 ? 1 : 0;
    if (env_int("CSRC_GPU_GBUF", 1) != 0 && P.gather_lanes >= 1 && P.gather_lanes <= 8) {
        const int R = P.gather_nt / P.gather_lanes;
        if (P.gather_lanes == 1) {  // the one instantiated one-row-per-thread shape (gather_stage_fn)
            P.gather_u = 8;
            P.gather_nb = 1;
            // fp32: a 6-block bound (40 registers, no spills) over the unbounded 43-register form,
            // C5 0.415 vs 0.424 ms, C3/C4 unchanged (profiles/r01_sweep_gather_minb_l1.txt);
            // CSRC_GPU_GMINB=1 restores the unbounded form
            const int mb1 = minb_env < 0 ? (sizeof(T) == 4 ? 6 : 1) : minb_env;
            P.gather_minb = mb1 == 6 ? 6 : 1;  // the instantiated bounds of this shape
        }
        // staged x (pattern form): x windows of each row block come in by TMA with the values
        P.gather_xs = P.gather_pat && P.gather_lanes >= 2 && env_int("CSRC_GPU_GXS", 0) != 0 &&
                              setup_staged_x<T>(P, pat_off)
                          ? 1
                          : 0;
        int64_t cap = 0;
        for (int64_t b = 0; b < n; b += R) cap = std::max<int64_t>(cap, eptr[std::min<int64_t>(n, b + R)] - eptr[b]);
        if (cap <= 16384) {
            P.gather_cap = static_cast<int>(cap);
            const int smem = gather_stage_smem<T>(P);
            if (smem <= 100 * 1024) {
                void* fn = gather_stage_fn<T>(P);
                set_smem_limit(reinterpret_cast<const void*>(fn), smem);
                // shared/L1 split: the driver's choice by default (L1 serves the x gathers)
                const int carve = env_int("CSRC_GPU_GCARVE", -1);
                if (carve >= 0)
                    CUDA_OK(cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, carve));
                int occ = 0;
                CUDA_OK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, P.gather_nt, smem));
                if (occ >= 1) {
                    P.gather_buf = 1;
                    const int64_t blocks = (n + R - 1) / R;
                    P.gather_grid = static_cast<int>(
                        std::min<int64_t>(blocks, static_cast<int64_t>(num_sms(P.device)) * occ));
                }
            }
        }
    }
    // sliced form for rows longer than ~40 entries with a small pattern dictionary
    // (C4 elasticity: 281 us vs 365 us staged); the staged form stays ahead on
    // 27-point rows (C5: 694 vs 705 us f64, 466 vs 565 us f32) and on explicit
    // columns (C3) -- profiles/r01_sweep_sell3.txt. CSRC_GPU_GSELL=0/1 forces.
    const int sell_env = env_int("CSRC_GPU_GSELL", -1);
    const bool sell_auto = has_pat && avg > 40.0;  // (not P.gather_pat: explicit columns keep the same form)
    mark("staged-kernel config");
    if ((sell_env == 1 || (sell_env < 0 && sell_auto)) && n > 0) {
        if (dv) {  // the sliced layout is built on the host: fetch the device-built values
            HostLink hl(P.stream);
            ev.resize(ne);
            hl.d2h(ev.data(), dv->ev.p, ne * 8);
            if (!value_symmetric) {
                evt.resize(ne);
                hl.d2h(evt.data(), dv->evt.p, ne * 8);
            }
        }
        setup_sell<T>(P, n, eptr, eidx, ev, evt, value_symmetric, pbase, pat_off);
        mark("sliced layout + upload");
        return;
    }
    upload(P.eptr, eptr.data(), eptr.size());
    if (dv) {  // values already on the device (build_entries_device)
        auto take = [&](DevBuf& dst, DevBuf& src) {
            if (std::is_same<T, double>::value) {
                adopt(dst, src);
            } else {
                dst.alloc(ne * sizeof(T));
                dev::k_convert<double, float><<<grid_for(P.device, static_cast<int64_t>(ne), 256), 256, 0,
                                                P.stream>>>(src.as<double>(), dst.as<float>(),
                                                            static_cast<int64_t>(ne));
                CUDA_OK(cudaGetLastError());
                CUDA_OK(cudaStreamSynchronize(P.stream));
            }
        };
        take(P.eval, dv->ev);
        if (!value_symmetric) take(P.eval_t, dv->evt);
    } else {
        upload_values<T>(P.eval, ev.data(), ev.size());
        if (!value_symmetric) upload_values<T>(P.eval_t, evt.data(), evt.size());
    }
    mark("value uploads");
    if (!P.gather_buf) P.gather_pat = 0;  // the plain row kernel reads explicit indices
    if (P.gather_pat) {
        upload(P.pbase, pbase.data(), pbase.size());
        upload(P.pat_off, pat_off.data(), pat_off.size());
    } else {
        P.n_patterns = 0;
        if (dv)
            adopt(P.eidx, dv->eidx);
        else
            upload(P.eidx, eidx.data(), eidx.size());
    }
}

// CSR plan (spmv_csr, kernels.hpp:7-22): the CSR rows are the entry stream
// as they stand (diagonal included, no ad term, no transposed stream).
template <class T>
void setup_gather_csr(Plan& P, index_t n_rows, index_t n_cols, const int32_t* rp, const int32_t* ci,
                      const double* va) {
    const int64_t nnz = rp[n_rows];
    std::vector<int32_t> eptr(rp, rp + n_rows + 1);
    HVec<int32_t> eidx(static_cast<size_t>(nnz));
    HVec<double> ev(static_cast<size_t>(nnz)), evt;
    parallel_slices(nnz, [&](int, int64_t b, int64_t e) {
        std::memcpy(eidx.data() + b, ci + b, static_cast<size_t>(e - b) * sizeof(int32_t));
        std::memcpy(ev.data() + b, va + b, static_cast<size_t>(e - b) * sizeof(double));
    });
    P.x_hi = n_cols;
    P.gi0 = P.gi1 = 0;
    // rectangular CSR: no host pipeline (its x chunks follow the rows)
    finish_gather<T>(P, n_rows, n_rows != n_cols, eptr, eidx, ev, evt, true,
                     env_int("CSRC_GPU_PLAN_TRACE", 0) != 0);
}

template <class T, int L, int PF>
void launch_gather_rows_LP(const Plan& P, const T* vals, const T* x, T* y, const int32_t* rows,
                           int32_t row0, int32_t count, cudaStream_t st) {
    const int64_t blocks = (static_cast<int64_t>(count) + 256 / L - 1) / (256 / L);
    const int64_t cap = static_cast<int64_t>(num_sms(P.device)) * std::max(1, P.gather_bpsm);
    const int grid = static_cast<int>(std::max<int64_t>(1, std::min(blocks, cap)));
    dev::k_gather_rows<T, L, PF><<<grid, 256, 0, st>>>(P.eptr.as<int32_t>(), P.eidx.as<int32_t>(),
                                                       vals, P.ad.as<T>(), x, y, rows, row0, count);
}

template <class T, int L>
void launch_gather_rows_L(const Plan& P, const T* vals, const T* x, T* y, int32_t r0, int32_t r1,
                          cudaStream_t st) {
    switch (P.gather_pf) {
        case 0: launch_gather_rows_LP<T, L, 0>(P, vals, x, y, nullptr, r0, r1 - r0, st); break;
        case 1: launch_gather_rows_LP<T, L, 1>(P, vals, x, y, nullptr, r0, r1 - r0, st); break;
        case 4: launch_gather_rows_LP<T, L, 4>(P, vals, x, y, nullptr, r0, r1 - r0, st); break;
        default: launch_gather_rows_LP<T, L, 2>(P, vals, x, y, nullptr, r0, r1 - r0, st); break;
    }
}

// rows [r0, r1) of the gather product (r0 a multiple of 256 / lanes unless 0)
template <class T>
void launch_gather_range(const Plan& P, bool tr, const T* x, T* y, int32_t r0, int32_t r1,
                         cudaStream_t st) {
    if (r1 <= r0) return;
    x += P.row_begin - P.lo;  // band plans: x holds [lo, x_hi), columns are band-row relative
    if (P.gather_sell) {
        dev::GSellArgs<T> A;
        A.sbase = P.sbase.as<int32_t>();
        A.rmeta = P.rmeta.as<int32_t>();
        A.sidx = P.sidx.as<int32_t>();
        A.pat_off = P.pat_off.as<int32_t>();
        A.sval = (tr && !P.value_symmetric ? P.sval_t : P.sval).template as<T>();
        A.ad = P.ad.as<T>();
        A.x = x;
        A.y = y;
        const int H = 32 / P.sell_lanes;
        A.slice0 = r0 / H;
        A.slice1 = (r1 + H - 1) / H;
        A.nrows = r1;
        A.pat_len = P.sell_pat_len;
        const int64_t blocks = (static_cast<int64_t>(A.slice1 - A.slice0) + 7) / 8;
        const int grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(blocks, P.sell_grid)));
        void* args[] = {&A};
        // the smem limit is an attribute of the kernel instantiation, shared by every plan of
        // this shape: set it per launch so a smaller plan created later cannot lower it
        set_smem_limit(sell_fn<T>(P), 4 * P.sell_pat_len);
        CUDA_OK(cudaLaunchKernel(sell_fn<T>(P), dim3(grid), dim3(256), args, static_cast<size_t>(4 * P.sell_pat_len),
                                 st));
        return;
    }
    const T* vals = (tr && !P.value_symmetric ? P.eval_t : P.eval).template as<T>();
    if (P.gather_buf) {
        const int R = P.gather_nt / P.gather_lanes;
        dev::GStageArgs<T> A;
        A.eptr = P.eptr.as<int32_t>();
        A.eidx = P.eidx.as<int32_t>();
        A.pbase = P.pbase.as<int32_t>();
        A.pat_off = P.pat_off.as<int32_t>();
        A.eval = vals;
        A.ad = P.ad.as<T>();
        A.x = x;
        A.y = y;
        A.row0 = r0;
        A.nrows = r1;
        A.idx_bytes = P.gather_pat ? 0 : dev::gather_idx_bytes(P.gather_cap);
        A.val_bytes = dev::gather_val_bytes<T>(P.gather_cap);
        A.xs_tab = nullptr;
        A.clo = A.chi = A.cbase = nullptr;
        A.n_clusters = 0;
        A.x_min = P.lo - P.row_begin;  // x holds [lo, x_hi) global = these kernel coordinates
        A.x_max = P.x_hi - P.row_begin;
        A.xs_bytes = 0;
        A.rs_bytes = gather_rs_bytes(P);
        if (P.gather_xs) {
            const int m = 16 / static_cast<int>(sizeof(T));
            const int ph = static_cast<int>((reinterpret_cast<uintptr_t>(x) / sizeof(T)) % m);
            A.xs_tab = P.xs_tab.as<int32_t>() + static_cast<size_t>(ph) * P.xs_tab_len;
            A.clo = P.xs_clo.as<int32_t>();
            A.chi = P.xs_chi.as<int32_t>();
            A.cbase = P.xs_cbase.as<int32_t>();
            A.n_clusters = P.xs_clusters;
            A.xs_bytes = P.xs_bytes;
        }
        const int64_t blocks = (static_cast<int64_t>(r1 - r0) + R - 1) / R;
        const int grid = static_cast<int>(std::min<int64_t>(blocks, P.gather_grid));
        void* args[] = {&A};
        set_smem_limit(gather_stage_fn<T>(P), gather_stage_smem<T>(P));  // per launch, as above
        CUDA_OK(cudaLaunchKernel(gather_stage_fn<T>(P), dim3(grid), dim3(P.gather_nt), args,
                                 static_cast<size_t>(gather_stage_smem<T>(P)), st));
        return;
    }
    switch (P.gather_lanes) {
        case 1: launch_gather_rows_L<T, 1>(P, vals, x, y, r0, r1, st); break;
        case 2: launch_gather_rows_L<T, 2>(P, vals, x, y, r0, r1, st); break;
        case 8: launch_gather_rows_L<T, 8>(P, vals, x, y, r0, r1, st); break;
        case 16: launch_gather_rows_L<T, 16>(P, vals, x, y, r0, r1, st); break;
        default: launch_gather_rows_L<T, 4>(P, vals, x, y, r0, r1, st); break;
    }
}

template <class T>
void launch_gather(const Plan& P, bool tr, const T* x, T* y, cudaStream_t st) {
    launch_gather_range<T>(P, tr, x, y, 0, P.nrows, st);
}

// -------------------------------------------------------------- creation
struct CreateOpts {
    const int32_t* color = nullptr;
    int32_t n_colors = 0;
    const int32_t* block_start = nullptr;
    int32_t bands = 0;
    bool band = false;
    index_t row_begin = 0, row_end = 0;
    // rectangular tail (csrc_gpu_plan_create_rect)
    int32_t m_cols = 0;
    const int32_t* rect_ptr = nullptr;
    const int32_t* rect_col = nullptr;
    const double* rect_val = nullptr;
};

template <class T>
void create_typed(Plan& P, const MatView& a, const csrc_gpu_strategy& s, const CreateOpts& o) {
    const index_t r0 = P.row_begin, r1 = P.row_end;
    const count_t t0 = a.ia[r0], t1 = a.ia[r1];
    P.k = t1 - t0;
    P.nrows = r1 - r0;
    P.value_symmetric = a.value_symmetric;
    P.nnz_stored = a.nnz_stored();
    P.sub_lanes = pick_lanes(P.k, P.nrows);
    // device arrays (band rows only)
    {
        std::vector<int32_t> ia_loc(static_cast<size_t>(P.nrows) + 1);
        for (index_t r = 0; r <= P.nrows; ++r) ia_loc[r] = a.ia[r0 + r] - static_cast<int32_t>(t0);
        upload(P.ia, ia_loc.data(), ia_loc.size());
    }
    const bool colored = P.exec_kind == CSRC_KIND_COLORFUL;
    const bool gather = P.exec_kind == CSRC_KIND_GATHER;  // keeps its own entry stream
    if (!colored && !gather) {
        upload(P.ja, a.ja + t0, static_cast<size_t>(P.k));
        upload_values<T>(P.al, a.al + t0, static_cast<size_t>(P.k));
        if (!a.value_symmetric) upload_values<T>(P.au, a.au + t0, static_cast<size_t>(P.k));
    }
    if (!colored) upload_values<T>(P.ad, a.ad + r0, static_cast<size_t>(P.nrows));
    if (o.m_cols) {
        P.m_cols = o.m_cols;
        P.rect_nnz = o.rect_ptr[a.n];
        std::vector<int32_t> gcol(static_cast<size_t>(P.rect_nnz));
        for (count_t q = 0; q < P.rect_nnz; ++q) gcol[q] = a.n + o.rect_col[q];
        upload(P.rt_ptr, o.rect_ptr, static_cast<size_t>(a.n) + 1);
        upload(P.rt_col, gcol.data(), gcol.size());
        upload_values<T>(P.rt_val, o.rect_val, static_cast<size_t>(P.rect_nnz));
    }
    switch (P.exec_kind) {
        case CSRC_KIND_WINDOWED: {
            std::vector<index_t> bs;
            if (o.block_start) bs.assign(o.block_start, o.block_start + o.bands + 1);
            setup_windowed<T>(P, a, o.block_start ? &bs : nullptr, s.bands,
                              o.block_start != nullptr);
            P.launches = 2;
            break;
        }
        case CSRC_KIND_LOCAL_BUFFERS: {
            std::vector<index_t> bs;
            if (o.block_start) bs.assign(o.block_start, o.block_start + o.bands + 1);
            setup_buffers<T>(P, a, o.block_start ? &bs : nullptr, s.bands);
            P.launches = 3;
            break;
        }
        case CSRC_KIND_COLORFUL: {
            std::vector<int32_t> color;
            int nc = 0;
            if (o.color) {
                color.assign(o.color, o.color + a.n);
                nc = o.n_colors;
            } else {
                color = color_rows(a, s.conflict_mode, s.color_order, &nc);
            }
            Validity v = validate_coloring(a, color.data(), nc);
            if (!v.valid)
                throw Error("coloring violation: rows " + std::to_string(v.row_a) + " and " +
                            std::to_string(v.row_b) + " both write y[" +
                            std::to_string(v.position) + "]");
            setup_colored<T>(P, a, color, nc);
            P.host_color = std::move(color);
            P.launches = P.cw ? 2 : 1 + nc;  // wave: counter memset + one persistent kernel
            break;
        }
        case CSRC_KIND_ATOMIC:
            P.launches = 2;
            break;
        case CSRC_KIND_GATHER:
            setup_gather<T>(P, a);
            P.launches = 1;
            break;
        default:
            throw Error("unknown strategy kind " + std::to_string(P.exec_kind));
    }
}

Plan* create_plan(const csrc_host_matrix* m, const csrc_gpu_strategy* s, const CreateOpts& o) {
    if (!s) throw Error("null strategy");
    const bool trace = env_int("CSRC_GPU_PLAN_TRACE", 0) != 0;
    const auto t_start = std::chrono::steady_clock::now();
    auto since = [&] {
        return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_start).count();
    };
    MatView a = view_of(m, true);
    if (trace) std::fprintf(stderr, "plan: structure check           %8.1f ms\n", since());
    // ParallelSpmv ctor checks (parallel.hpp:229-234)
    if (s->p < 1) throw Error("ParallelSpmv: thread count must be >= 1");
    if (s->kind == CSRC_KIND_SEQUENTIAL && s->p != 1)
        throw Error("ParallelSpmv: sequential strategy requires p = 1");
    if (s->kind < CSRC_KIND_SEQUENTIAL || s->kind > CSRC_KIND_GATHER)
        throw Error("unknown strategy kind " + std::to_string(s->kind));
    if (s->dtype != CSRC_DTYPE_F64 && s->dtype != CSRC_DTYPE_F32)
        throw Error("unknown dtype " + std::to_string(s->dtype));
    if (s->kind == CSRC_KIND_LOCAL_BUFFERS &&
        (s->accum < CSRC_ACCUM_ALL_IN_ONE || s->accum > CSRC_ACCUM_INTERVAL))
        throw Error("unknown accumulation method " + std::to_string(s->accum));
    if (o.color && s->kind != CSRC_KIND_COLORFUL)
        throw Error("ParallelSpmv: colorful plan given to a different strategy");
    if (o.block_start) {
        if (s->kind != CSRC_KIND_LOCAL_BUFFERS && s->kind != CSRC_KIND_WINDOWED)
            throw Error("ParallelSpmv: local-buffers plan given to a different strategy");
        if (s->kind == CSRC_KIND_LOCAL_BUFFERS && s->p >= 2 && o.bands != s->p)
            throw Error("ParallelSpmv: plan built for p=" + std::to_string(o.bands) +
                        ", strategy has p=" + std::to_string(s->p));
        if (o.bands < 1 || o.block_start[0] != 0 || o.block_start[o.bands] != a.n)
            throw Error("partition must cover rows [0, n)");
        for (int b = 0; b < o.bands; ++b)
            if (o.block_start[b + 1] <= o.block_start[b])
                throw Error("effective_range: empty block");
    }
    if (o.color) {
        if (o.n_colors < 1 && a.n > 0) throw Error("coloring has no classes");
        for (index_t i = 0; i < a.n; ++i)
            if (o.color[i] < 0 || o.color[i] >= o.n_colors)
                throw Error("coloring: row " + std::to_string(i) + " colour out of range");
    }
    if (o.m_cols) {
        if (o.band) throw Error("band plans take square matrices only");
        if (o.m_cols <= a.n)
            throw Error("ParallelSpmv: rectangular matrix needs m > n (got m=" + std::to_string(o.m_cols) +
                        ", n=" + std::to_string(a.n) + ")");
        if (!o.rect_ptr || o.rect_ptr[0] != 0) throw Error("rect tail: row_ptr must start at 0");
        for (index_t i = 0; i < a.n; ++i)
            if (o.rect_ptr[i + 1] < o.rect_ptr[i]) throw Error("rect tail: row_ptr must be non-decreasing");
        const count_t tn = o.rect_ptr[a.n];
        if (tn > 0 && (!o.rect_col || !o.rect_val)) throw Error("rect tail: null column or value array");
        for (count_t q = 0; q < tn; ++q)
            if (o.rect_col[q] < 0 || o.rect_col[q] >= o.m_cols - a.n)
                throw Error("rect tail: column " + std::to_string(o.rect_col[q]) + " outside [0, " +
                            std::to_string(o.m_cols - a.n) + ")");
    }
    auto P = std::make_unique<Plan>();
    P->device = s->device;
    CUDA_OK(cudaSetDevice(P->device));
    P->kind = s->kind;
    P->accum = s->accum;
    P->dtype = s->dtype;
    P->p_ref = s->p;
    P->n_global = a.n;
    if (o.band) {
        if (o.row_begin < 0 || o.row_end > a.n || o.row_begin >= o.row_end)
            throw Error("band rows must satisfy 0 <= row_begin < row_end <= n");
        P->row_begin = o.row_begin;
        P->row_end = o.row_end;
        index_t lo = o.row_begin;
        for (index_t t = a.ia[o.row_begin]; t < a.ia[o.row_end]; ++t) lo = std::min(lo, a.ja[t]);
        P->lo = lo;
    } else {
        P->row_begin = 0;
        P->row_end = a.n;
        P->lo = 0;
    }
    // what runs: p = 1 or sequential short-circuit (parallel.hpp:197-202) -> no buffers;
    // the gather kernel (deterministic, fastest) for whole-matrix plans, windowed for bands
    P->exec_kind = s->kind;
    const int single = o.band ? CSRC_KIND_WINDOWED : CSRC_KIND_GATHER;
    if (s->kind == CSRC_KIND_SEQUENTIAL) P->exec_kind = single;
    if (s->kind == CSRC_KIND_LOCAL_BUFFERS && s->p < 2 && !o.block_start) P->exec_kind = single;
    if (o.band && (P->exec_kind == CSRC_KIND_LOCAL_BUFFERS || P->exec_kind == CSRC_KIND_COLORFUL))
        throw Error("band plans support the windowed, atomic and gather kernels only");
    CUDA_OK(cudaStreamCreateWithFlags(&P->stream, cudaStreamNonBlocking));
    for (auto& e : P->ev) CUDA_OK(cudaEventCreate(&e));
    if (a.n == 0) return P.release();
    if (trace) std::fprintf(stderr, "plan: streams + events          %8.1f ms\n", since());
    if (P->dtype == CSRC_DTYPE_F64)
        create_typed<double>(*P, a, *s, o);
    else
        create_typed<float>(*P, a, *s, o);
    if (trace) std::fprintf(stderr, "plan: total in the library      %8.1f ms\n", since());
    return P.release();
}

// --------------------------------------------------------------- apply
int grid_for(int device, int64_t work, int per_block) {
    int64_t blocks = (work + per_block - 1) / per_block;
    const int64_t cap = static_cast<int64_t>(num_sms(device)) * 16;
    return static_cast<int>(std::max<int64_t>(1, std::min(blocks, cap)));
}

template <class T, int L>
void launch_atomic_L(const Plan& P, const T* al, const T* au, const T* x, T* y, cudaStream_t st) {
    const int rows_per_block = 256 / L;
    dev::k_atomic<T, L><<<grid_for(P.device, P.nrows, rows_per_block), 256, 0, st>>>(
        P.ia.as<int32_t>(), P.ja.as<int32_t>(), al, au, P.ad.as<T>(), x, y, P.nrows,
        P.row_begin, -static_cast<int64_t>(P.lo));
}

template <class T, int L>
void launch_colored_L(const Plan& P, const T* al, const T* au, const T* x, T* y,
                      cudaStream_t st) {
    for (int c = 0; c < P.n_colors; ++c) {
        const count_t c0 = P.class_ptr[c], c1 = P.class_ptr[c + 1];
        if (c1 <= c0) continue;
        dev::k_colored<T, L><<<grid_for(P.device, c1 - c0, 256 / L), 256, 0, st>>>(
            P.rid.as<int32_t>(), P.cia.as<int64_t>(), P.cja.as<int32_t>(), al, au,
            P.cad.as<T>(), x, y, c0, c1, -static_cast<int64_t>(P.lo));
    }
}

template <class T>
void launch_atomic(const Plan& P, bool tr, const T* x, T* y, cudaStream_t st) {
    const T* al = (tr ? P.au : P.al).template as<T>();
    const T* au = (tr ? P.al : P.au).template as<T>();
    if (P.value_symmetric) au = al = P.al.as<T>();
    switch (P.sub_lanes) {
        case 2: launch_atomic_L<T, 2>(P, al, au, x, y, st); break;
        case 4: launch_atomic_L<T, 4>(P, al, au, x, y, st); break;
        case 8: launch_atomic_L<T, 8>(P, al, au, x, y, st); break;
        case 16: launch_atomic_L<T, 16>(P, al, au, x, y, st); break;
        default: launch_atomic_L<T, 32>(P, al, au, x, y, st); break;
    }
}

template <class T>
void launch_colored_ring(const Plan& P, bool tr, const T* x, T* y, cudaStream_t st) {
    dev::ColorRingArgs<T> A{};
    A.tickets = P.cw_tk.as<dev::CwTicket>();
    A.nch = P.cw_nch.as<int32_t>();
    A.ctr = P.cw_ctr.as<int32_t>();
    A.n_tickets = P.cw_tickets;
    A.n_blocks = P.cw_blocks;
    A.n_e = P.n_colors + 2;
    A.radius = P.cw_radius;
    A.rid = P.rid.as<int32_t>();
    A.pk = P.cpk.as<unsigned char>();
    A.ad = P.cad.as<T>();
    A.x = x;
    A.y = y;
    A.xp = P.cw_xp.as<T>();
    A.yp = P.cw_yp.as<T>();
    A.stages = P.cr_stages;
    A.stage_bytes = P.cr_stage_bytes;
    A.sym = P.value_symmetric ? 1 : 0;
    A.tr = tr ? 1 : 0;
    A.pf = P.cr_pf;
    A.claim = P.cr_claim;
    CUDA_OK(cudaMemsetAsync(P.cw_ctr.p, 0, static_cast<size_t>(P.cw_tasks + 1) * 4, st));
    const void* fn = colored_ring_fn<T>(P);
    const int smem = P.cr_stages * P.cr_stage_bytes;
    set_smem_limit(fn, smem);
    void* args[] = {&A};
    CUDA_OK(cudaLaunchKernel(fn, dim3(P.cw_grid), dim3(colored_ring_threads(P)), args, smem, st));
}

template <class T>
void launch_colored_wave(const Plan& P, bool tr, const T* x, T* y, cudaStream_t st) {
    if (P.cw_ring) {
        launch_colored_ring<T>(P, tr, x, y, st);
        return;
    }
    dev::ColorWaveArgs<T> A{};
    A.tickets = P.cw_tk.as<dev::CwTicket>();
    A.nch = P.cw_nch.as<int32_t>();
    A.ctr = P.cw_ctr.as<int32_t>();
    A.n_tickets = P.cw_tickets;
    A.n_blocks = P.cw_blocks;
    A.n_e = P.n_colors + 2;
    A.radius = P.cw_radius;
    A.rid = P.rid.as<int32_t>();
    A.ja = P.cja.as<int32_t>();
    A.al = (tr ? P.cau : P.cal).template as<T>();
    A.au = (tr ? P.cal : P.cau).template as<T>();
    if (P.value_symmetric) A.au = A.al = P.cal.as<T>();
    A.ad = P.cad.as<T>();
    A.x = x;
    A.y = y;
    A.xp = P.cw_xp.as<T>();
    A.yp = P.cw_yp.as<T>();
    A.pf_mode = P.cw_pf;
    // ticket counter + per-task completion counts start at zero every product
    CUDA_OK(cudaMemsetAsync(P.cw_ctr.p, 0, static_cast<size_t>(P.cw_tasks + 1) * 4, st));
    void* args[] = {&A};
    CUDA_OK(cudaLaunchKernel(colored_wave_fn<T>(P), dim3(P.cw_grid), dim3(P.cw_nt), args, 0, st));
}

template <class T>
void launch_colored(const Plan& P, bool tr, const T* x, T* y, cudaStream_t st) {
    if (P.cw) {
        launch_colored_wave<T>(P, tr, x, y, st);
        return;
    }
    const T* al = (tr ? P.cau : P.cal).template as<T>();
    const T* au = (tr ? P.cal : P.cau).template as<T>();
    if (P.value_symmetric) au = al = P.cal.as<T>();
    switch (P.sub_lanes) {
        case 2: launch_colored_L<T, 2>(P, al, au, x, y, st); break;
        case 4: launch_colored_L<T, 4>(P, al, au, x, y, st); break;
        case 8: launch_colored_L<T, 8>(P, al, au, x, y, st); break;
        case 16: launch_colored_L<T, 16>(P, al, au, x, y, st); break;
        default: launch_colored_L<T, 32>(P, al, au, x, y, st); break;
    }
}

template <class T>
void launch_windowed(const Plan& P, dev::WinArgs<T> A, int ctas, cudaStream_t st) {
    if (ctas <= 0) return;
    if (P.value_symmetric) A.au = A.al;
    auto fn = windowed_fn<T>(P.win_lanes, P.tile_rows, P.win_ring);
    // per-plan shared-memory size: the attribute is per function, so set it per launch
    set_smem_limit(reinterpret_cast<const void*>(fn), static_cast<int>(P.win_smem));
    fn<<<ctas, 32 + P.tile_rows * P.win_lanes, P.win_smem, st>>>(A);
}

void rec(const Plan& P, int i, cudaStream_t st) {
    if (P.timing) CUDA_OK(cudaEventRecord(P.ev[i], st));
}

template <class T>
void apply_typed(Plan& P, const void* dx, void* dy, cudaStream_t st, bool tr, int part) {
    const T* x = static_cast<const T*>(dx);
    T* y = static_cast<T*>(dy);
    const size_t ybytes = static_cast<size_t>(P.vec_len()) * sizeof(T);
    if (part >= 0) {
        if (P.exec_kind != CSRC_KIND_WINDOWED)
            throw Error("boundary / interior parts need a windowed band plan");
        // band plan partial products
        if (part == 0) CUDA_OK(cudaMemsetAsync(y, 0, ybytes, st));
        auto A = win_args<T>(P, dx, dy, tr);
        A.tiles = P.sched_part[part].as<dev::TileDesc>();
        A.cta_ptr = P.cta_ptr_part[part].as<int32_t>();
        launch_windowed<T>(P, A, P.bands_part[part], st);
        CUDA_OK(cudaGetLastError());
        return;
    }
    rec(P, 0, st);
    switch (P.exec_kind) {
        case CSRC_KIND_WINDOWED: {
            CUDA_OK(cudaMemsetAsync(y, 0, ybytes, st));
            rec(P, 1, st);
            launch_windowed<T>(P, win_args<T>(P, dx, dy, tr), P.bands, st);
            rec(P, 2, st);
            break;
        }
        case CSRC_KIND_ATOMIC: {
            CUDA_OK(cudaMemsetAsync(y, 0, ybytes, st));
            rec(P, 1, st);
            launch_atomic<T>(P, tr, x, y, st);
            rec(P, 2, st);
            break;
        }
        case CSRC_KIND_GATHER: {
            rec(P, 1, st);  // no init: every y element is written once
            launch_gather<T>(P, tr, x, y, st);
            rec(P, 2, st);
            break;
        }
        case CSRC_KIND_COLORFUL: {
            if (!P.cw) CUDA_OK(cudaMemsetAsync(y, 0, ybytes, st));  // the wave zeroes its own y
            rec(P, 1, st);
            launch_colored<T>(P, tr, x, y, st);
            rec(P, 2, st);
            break;
        }
        case CSRC_KIND_LOCAL_BUFFERS: {
            // init: y (the owner parts of the buffers) and the spill buffers
            auto B = buf_args<T>(P);
            const int sms = num_sms(P.device);
            CUDA_OK(cudaMemsetAsync(y, 0, ybytes, st));
            if (P.buf_total > 0) {
                switch (P.accum) {
                    case CSRC_ACCUM_ALL_IN_ONE:
                        dev::k_init_flat<T><<<grid_for(P.device, P.buf_total, 256), 256, 0, st>>>(
                            B.spill, P.buf_total);
                        break;
                    case CSRC_ACCUM_PER_BUFFER:
                    case CSRC_ACCUM_EFFECTIVE: {
                        dim3 g(std::max(1, sms * 4 / std::max(1, P.lb_bands)), std::min(P.lb_bands, 65535));
                        dev::k_init_per_buffer<T><<<g, 256, 0, st>>>(B);
                        break;
                    }
                    default: {
                        dim3 g(std::max(1, sms * 4 / std::max(1, P.n_iv)), std::min(std::max(P.n_iv, 1), 65535));
                        dev::k_init_interval<T><<<g, 256, 0, st>>>(B);
                    }
                }
            }
            rec(P, 1, st);
            // compute: the wavefront windowed kernel, out-of-band scatters to the spills
            auto A = win_args<T>(P, dx, dy, tr);
            A.tile_band = P.tile_band.as<int32_t>();
            A.band_rs = P.band_rs.as<int32_t>();
            A.spill_shift = P.spill_shift.as<int64_t>();
            A.spill = B.spill;
            launch_windowed<T>(P, A, P.bands, st);
            rec(P, 2, st);
            // accumulate: y[q] += covering spills, ascending band id
            const int64_t shift = -static_cast<int64_t>(P.lo);
            if (P.buf_total > 0) {
                switch (P.accum) {
                    case CSRC_ACCUM_ALL_IN_ONE:
                    case CSRC_ACCUM_PER_BUFFER: {
                        dim3 g(4, std::min(std::max(P.lb_bands, 1) * 8, 65535));
                        dev::k_accum_sliced<T><<<g, 256, 0, st>>>(B, y, P.row_begin, P.row_end, shift);
                        break;
                    }
                    case CSRC_ACCUM_EFFECTIVE: {
                        dim3 g(std::max(1, sms * 2 / std::max(1, P.lb_bands)), std::min(P.lb_bands, 65535));
                        dev::k_accum_effective<T><<<g, 256, 0, st>>>(B, y, shift);
                        break;
                    }
                    default: {
                        dim3 g(std::max(1, sms * 2 / std::max(1, P.n_iv)), std::min(std::max(P.n_iv, 1), 65535));
                        dev::k_accum_interval<T><<<g, 256, 0, st>>>(B, y, shift);
                    }
                }
            }
            break;
        }
        default:
            throw Error("unknown strategy kind");
    }
    if (P.m_cols) {
        if (tr) throw Error("spmv_csrc_transpose: rectangular plans have no transpose product");
        dev::k_rect_tail<T, 4><<<grid_for(P.device, P.nrows, 64), 256, 0, st>>>(
            P.rt_ptr.as<int32_t>(), P.rt_col.as<int32_t>(), P.rt_val.as<T>(), x, y, P.nrows);
    }
    rec(P, 3, st);
    P.ev_recorded = P.timing;
    CUDA_OK(cudaGetLastError());
}

// Products that touch plan-owned scratch (local-buffers band buffers, the timing
// events, the colored plan's class-order vectors) on a caller stream other than
// the plan's own are ordered both ways against the plan's stream, so host
// applies / time_products (plan stream) and apply_device (caller stream) on one
// plan never overlap on that scratch. Skipped while the caller's stream is
// capturing a graph (the capture orders itself).
struct StreamJoin {
    Plan& P;
    cudaStream_t st;
    bool on = false;
    StreamJoin(Plan& p, cudaStream_t s, bool uses_scratch) : P(p), st(s) {
        if (!uses_scratch || st == P.stream) return;
        cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
        CUDA_OK(cudaStreamIsCapturing(st, &cs));
        if (cs != cudaStreamCaptureStatusNone) return;
        for (auto& e : P.ev_join)
            if (!e) CUDA_OK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        CUDA_OK(cudaEventRecord(P.ev_join[0], P.stream));
        CUDA_OK(cudaStreamWaitEvent(st, P.ev_join[0], 0));
        on = true;
    }
    void done() {
        if (!on) return;
        CUDA_OK(cudaEventRecord(P.ev_join[1], st));
        CUDA_OK(cudaStreamWaitEvent(P.stream, P.ev_join[1], 0));
    }
};

bool uses_plan_scratch(const Plan& P) {
    return P.timing || P.exec_kind == CSRC_KIND_LOCAL_BUFFERS || P.exec_kind == CSRC_KIND_COLORFUL;
}

void apply_device(Plan& P, const void* dx, void* dy, cudaStream_t st, bool tr, int part = -1) {
    if (tr && P.is_csr) throw Error("spmv_csr: CSR plans have no transpose product");
    if (P.nrows == 0) return;
    CUDA_OK(cudaSetDevice(P.device));
    StreamJoin join(P, st, uses_plan_scratch(P));
    if (P.dtype == CSRC_DTYPE_F64)
        apply_typed<double>(P, dx, dy, st, tr, part);
    else
        apply_typed<float>(P, dx, dy, st, tr, part);
    join.done();
}

// Host product with the copies overlapped (gather plans): x goes up in row
// chunks on s_h2d; chunk c's rows run on the compute stream once the last x
// chunk they read (hneed[c], plan time) has landed; its y rows go down on
// s_d2h while later chunks compute. H2D and D2H use the two copy directions
// of the link concurrently. Same kernels and summation order as the device
// entry point, so results are bit-identical to it.
// Pinned staging for pageable host vectors (lazily, once per plan).
void ensure_staging(Plan& P, bool x_stage, bool y_stage) {
    if ((x_stage || y_stage) && !P.cpool) {
        const int hw = static_cast<int>(std::max(1u, std::thread::hardware_concurrency()));
        P.cpool = std::make_unique<CopyPool>(std::min(hw, 16));
    }
    if (x_stage && !P.hx_pin)
        CUDA_OK(cudaHostAlloc(reinterpret_cast<void**>(&P.hx_pin), static_cast<size_t>(P.x_len()) * 8,
                              cudaHostAllocDefault));
    if (y_stage && !P.hy_pin)
        CUDA_OK(cudaHostAlloc(reinterpret_cast<void**>(&P.hy_pin), static_cast<size_t>(P.n_global) * 8,
                              cudaHostAllocDefault));
}

// Host product with the copies overlapped (gather plans): x goes up in row
// chunks on s_h2d; chunk c's rows run on the compute stream once the last x
// chunk they read (hneed[c], plan time) has landed; its y rows go down on
// s_d2h while later chunks compute. H2D and D2H use the two copy directions
// of the link concurrently. Pageable x / y (the reference API's std::vector)
// are staged through pinned buffers by the copy pool inside the same chunk
// loop: chunk c+1 of x is copied while chunk c is on the link, and finished y
// chunks are copied out while later x chunks still stage. Same kernels and
// summation order as the device entry point, so results are bit-identical.
void apply_host_pipelined(Plan& P, const double* xh, double* yh, bool tr) {
    const int nc = static_cast<int>(P.hchunk.size()) - 1;
    if (!P.s_h2d) {
        CUDA_OK(cudaStreamCreateWithFlags(&P.s_h2d, cudaStreamNonBlocking));
        CUDA_OK(cudaStreamCreateWithFlags(&P.s_d2h, cudaStreamNonBlocking));
        CUDA_OK(cudaStreamCreateWithFlags(&P.s_h2d2, cudaStreamNonBlocking));
        CUDA_OK(cudaStreamCreateWithFlags(&P.s_d2h2, cudaStreamNonBlocking));
        CUDA_OK(cudaEventCreateWithFlags(&P.ev_in, cudaEventDisableTiming));
        P.ev_x.assign(nc, nullptr);
        P.ev_y.assign(nc, nullptr);
        P.ev_d.assign(nc, nullptr);
        for (int c = 0; c < nc; ++c) {
            CUDA_OK(cudaEventCreateWithFlags(&P.ev_x[c], cudaEventDisableTiming));
            CUDA_OK(cudaEventCreateWithFlags(&P.ev_y[c], cudaEventDisableTiming));
            CUDA_OK(cudaEventCreateWithFlags(&P.ev_d[c], cudaEventDisableTiming));
        }
    }
    const bool xs = !host_pinned(xh), ys = !host_pinned(yh);
    ensure_staging(P, xs, ys);
    const double* xsrc = xs ? P.hx_pin : xh;
    double* ydst = ys ? P.hy_pin : yh;
    const bool f32 = P.dtype == CSRC_DTYPE_F32;
    if (f32) {
        const size_t n = static_cast<size_t>(P.n_global);
        if (!P.dxd.p) P.dxd.alloc(n * 8);
        if (!P.dyd.p) P.dyd.alloc(n * 8);
    }
    double* xd64 = f32 ? P.dxd.as<double>() : P.dx.as<double>();
    double* yd64 = f32 ? P.dyd.as<double>() : P.dy.as<double>();
    cudaStream_t st = P.stream;
    // CSRC_GPU_HOST_TRACE=1: per-chunk timeline on stderr (diagnostics only)
    const bool trace = env_int("CSRC_GPU_HOST_TRACE", 0) != 0;
    std::vector<cudaEvent_t> tr_ev;
    if (trace) {
        tr_ev.resize(1 + 3 * nc);
        for (auto& e : tr_ev) CUDA_OK(cudaEventCreate(&e));
        CUDA_OK(cudaEventRecord(tr_ev[0], st));
    }
    // CSRC_GPU_HOST_H2D_STREAMS / _D2H_STREAMS = 2: alternate chunks over two
    // copy streams per direction (diagnostics; default one each)
    const bool h2d2 = env_int("CSRC_GPU_HOST_H2D_STREAMS", 1) == 2;
    const bool d2h2 = env_int("CSRC_GPU_HOST_D2H_STREAMS", 1) == 2;
    CUDA_OK(cudaEventRecord(P.ev_in, st));
    CUDA_OK(cudaStreamWaitEvent(P.s_h2d, P.ev_in, 0));  // after earlier work on the plan stream
    if (h2d2) CUDA_OK(cudaStreamWaitEvent(P.s_h2d2, P.ev_in, 0));
    // CSRC_GPU_HOST_GRID_DIV=d: chunk products on 1/d of the usual grid (diagnostics: leaves HBM
    // headroom for the copy engines' writes while the link is the bottleneck)
    const int grid_div = std::max(1, env_int("CSRC_GPU_HOST_GRID_DIV", 1));
    struct GridRestore {
        Plan& p;
        int g, s;
        ~GridRestore() { p.gather_grid = g, p.sell_grid = s; }
    } restore{P, P.gather_grid, P.sell_grid};
    P.gather_grid = std::max(1, P.gather_grid / grid_div);
    P.sell_grid = std::max(1, P.sell_grid / grid_div);
    int have = -1;  // x chunks the compute stream already waited for (and converted)
    auto compute_chunk = [&](int c) {
        for (; have < P.hneed[c]; ++have) {
            CUDA_OK(cudaStreamWaitEvent(st, P.ev_x[have + 1], 0));
            if (f32) {
                const int32_t a = P.xchunk[have + 1], b = P.xchunk[have + 2];
                dev::k_convert<double, float><<<grid_for(P.device, b - a, 256), 256, 0, st>>>(
                    P.dxd.as<double>() + a, P.dx.as<float>() + a, b - a);
            }
        }
        const int32_t r0 = P.hchunk[c], r1 = P.hchunk[c + 1];
        if (f32) {
            launch_gather_range<float>(P, tr, P.dx.as<float>(), P.dy.as<float>(), r0, r1, st);
            dev::k_convert<float, double><<<grid_for(P.device, r1 - r0, 256), 256, 0, st>>>(
                P.dy.as<float>() + r0, P.dyd.as<double>() + r0, r1 - r0);
        } else {
            launch_gather_range<double>(P, tr, P.dx.as<double>(), P.dy.as<double>(), r0, r1, st);
        }
        CUDA_OK(cudaGetLastError());
        CUDA_OK(cudaEventRecord(P.ev_y[c], st));
        if (trace) CUDA_OK(cudaEventRecord(tr_ev[1 + nc + c], st));
        cudaStream_t sd = d2h2 && (c & 1) ? P.s_d2h2 : P.s_d2h;
        CUDA_OK(cudaStreamWaitEvent(sd, P.ev_y[c], 0));
        CUDA_OK(cudaMemcpyAsync(ydst + r0, yd64 + r0, static_cast<size_t>(r1 - r0) * 8,
                                cudaMemcpyDeviceToHost, sd));
        CUDA_OK(cudaEventRecord(P.ev_d[c], sd));
        if (trace) CUDA_OK(cudaEventRecord(tr_ev[1 + 2 * nc + c], sd));
    };
    int next_c = 0, next_out = 0;  // chunks enqueued for compute / copied out to a pageable y
    auto copy_out = [&](bool block) {
        for (; next_out < next_c; ++next_out) {
            if (block)
                CUDA_OK(cudaEventSynchronize(P.ev_d[next_out]));
            else if (cudaEventQuery(P.ev_d[next_out]) != cudaSuccess)
                break;
            const size_t r0 = P.hchunk[next_out], len = P.hchunk[next_out + 1] - P.hchunk[next_out];
            P.cpool->copy(yh + r0, P.hy_pin + r0, len * 8);
        }
    };
    for (int c = 0; c < nc; ++c) {
        const size_t r0 = P.xchunk[c], len = P.xchunk[c + 1] - P.xchunk[c];
        if (xs) P.cpool->copy(P.hx_pin + r0, xh + r0, len * 8);
        cudaStream_t sc = h2d2 && (c & 1) ? P.s_h2d2 : P.s_h2d;
        CUDA_OK(cudaMemcpyAsync(xd64 + r0, xsrc + r0, len * 8, cudaMemcpyHostToDevice, sc));
        CUDA_OK(cudaEventRecord(P.ev_x[c], sc));
        if (trace) CUDA_OK(cudaEventRecord(tr_ev[1 + c], sc));
        for (; next_c < nc && P.hneed[next_c] <= c; ++next_c) compute_chunk(next_c);
        if (ys) copy_out(false);
    }
    for (; next_c < nc; ++next_c) compute_chunk(next_c);
    if (ys) copy_out(true);
    CUDA_OK(cudaStreamSynchronize(P.s_d2h));
    if (d2h2) CUDA_OK(cudaStreamSynchronize(P.s_d2h2));
    if (h2d2) CUDA_OK(cudaStreamSynchronize(P.s_h2d2));
    CUDA_OK(cudaStreamSynchronize(st));
    if (trace) {
        std::fprintf(stderr, "host pipeline: %d chunks (ms from start: x landed / rows done / y landed)\n", nc);
        for (int c = 0; c < nc; ++c) {
            float a = 0, b = 0, d = 0;
            cudaEventElapsedTime(&a, tr_ev[0], tr_ev[1 + c]);
            cudaEventElapsedTime(&b, tr_ev[0], tr_ev[1 + nc + c]);
            cudaEventElapsedTime(&d, tr_ev[0], tr_ev[1 + 2 * nc + c]);
            std::fprintf(stderr, "  chunk %2d rows %9d..%9d need x<=%2d : %7.3f %7.3f %7.3f\n", c,
                         P.hchunk[c], P.hchunk[c + 1], P.hneed[c], a, b, d);
        }
        for (auto e : tr_ev) cudaEventDestroy(e);
    }
}

void apply_host(Plan& P, const double* xh, int64_t x_len, double* yh, bool tr) {
    if (x_len != P.x_len())
        throw Error(std::string(P.is_csr ? "spmv_csr" : "ParallelSpmv") + ": x has length " + std::to_string(x_len) +
                    ", expected " + std::to_string(P.x_len()));
    if (P.row_begin != 0 || P.row_end != P.n_global)
        throw Error("host products need a full-matrix plan (use the device entry points for bands)");
    if (P.n_global == 0) return;
    CUDA_OK(cudaSetDevice(P.device));
    const size_t n = static_cast<size_t>(P.n_global);
    const size_t nx = static_cast<size_t>(P.x_len());
    if (!P.dx.p) P.dx.alloc(nx * P.vsize());
    if (!P.dy.p) P.dy.alloc(n * P.vsize());
    cudaStream_t st = P.stream;
    if (P.exec_kind == CSRC_KIND_GATHER && P.hchunk.size() > 2 && !P.timing && !P.m_cols) {
        apply_host_pipelined(P, xh, yh, tr);
        return;
    }
    // pageable x / y: whole-vector staging through the plan's pinned buffers
    const bool xs = !host_pinned(xh), ys = !host_pinned(yh);
    ensure_staging(P, xs, ys);
    double* const y_user = yh;
    if (xs) {
        P.cpool->copy(P.hx_pin, xh, nx * 8);
        xh = P.hx_pin;
    }
    if (ys) yh = P.hy_pin;
    if (P.dtype == CSRC_DTYPE_F64) {
        CUDA_OK(cudaMemcpyAsync(P.dx.p, xh, nx * 8, cudaMemcpyHostToDevice, st));
        apply_device(P, P.dx.p, P.dy.p, st, tr);
        CUDA_OK(cudaMemcpyAsync(yh, P.dy.p, n * 8, cudaMemcpyDeviceToHost, st));
    } else {
        if (!P.dxd.p) P.dxd.alloc(nx * 8);
        if (!P.dyd.p) P.dyd.alloc(n * 8);
        CUDA_OK(cudaMemcpyAsync(P.dxd.p, xh, nx * 8, cudaMemcpyHostToDevice, st));
        dev::k_convert<double, float><<<grid_for(P.device, nx, 256), 256, 0, st>>>(
            P.dxd.as<double>(), P.dx.as<float>(), nx);
        apply_device(P, P.dx.p, P.dy.p, st, tr);
        dev::k_convert<float, double><<<grid_for(P.device, n, 256), 256, 0, st>>>(
            P.dy.as<float>(), P.dyd.as<double>(), n);
        CUDA_OK(cudaMemcpyAsync(yh, P.dyd.p, n * 8, cudaMemcpyDeviceToHost, st));
    }
    CUDA_OK(cudaStreamSynchronize(st));
    if (ys) P.cpool->copy(y_user, P.hy_pin, n * 8);
}

Plan* create_csr_plan(int32_t n_rows, int32_t n_cols, const int32_t* rp, const int32_t* ci, const double* va,
                      const csrc_gpu_strategy* s) {
    if (!s) throw Error("null strategy");
    if (s->kind != CSRC_KIND_SEQUENTIAL && s->kind != CSRC_KIND_GATHER)
        throw Error("CSR plans run the gather kernel (strategy sequential or gather)");
    if (s->dtype != CSRC_DTYPE_F64 && s->dtype != CSRC_DTYPE_F32)
        throw Error("unknown dtype " + std::to_string(s->dtype));
    if (n_rows < 0 || n_cols < 0) throw Error("spmv_csr: negative dimensions");
    if (!rp || rp[0] != 0) throw Error("spmv_csr: row_ptr must start at 0");
    for (index_t i = 0; i < n_rows; ++i)
        if (rp[i + 1] < rp[i]) throw Error("spmv_csr: row_ptr not nondecreasing at row " + std::to_string(i));
    const int64_t nnz = rp[n_rows];
    if (nnz > 0 && (!ci || !va)) throw Error("spmv_csr: null column or value array");
    for (int64_t q = 0; q < nnz; ++q)
        if (ci[q] < 0 || ci[q] >= n_cols)
            throw Error("spmv_csr: column " + std::to_string(ci[q]) + " outside [0, " + std::to_string(n_cols) + ")");
    auto P = std::make_unique<Plan>();
    P->device = s->device;
    CUDA_OK(cudaSetDevice(P->device));
    P->kind = CSRC_KIND_GATHER;
    P->exec_kind = CSRC_KIND_GATHER;
    P->dtype = s->dtype;
    P->p_ref = s->p;
    P->n_global = n_rows;
    P->row_begin = 0;
    P->row_end = n_rows;
    P->lo = 0;
    P->nrows = n_rows;
    P->k = nnz;
    P->value_symmetric = true;  // one value stream: no transpose product for CSR plans
    P->is_csr = true;
    P->csr_cols = n_cols;
    P->launches = 1;
    CUDA_OK(cudaStreamCreateWithFlags(&P->stream, cudaStreamNonBlocking));
    for (auto& e : P->ev) CUDA_OK(cudaEventCreate(&e));
    if (n_rows == 0) return P.release();
    if (P->dtype == CSRC_DTYPE_F64)
        setup_gather_csr<double>(*P, n_rows, n_cols, rp, ci, va);
    else
        setup_gather_csr<float>(*P, n_rows, n_cols, rp, ci, va);
    return P.release();
}

Plan* checked(csrc_gpu_plan_t p) {
    if (!p) throw Error("null plan");
    return p;
}

}  // namespace

extern "C" {

int csrc_gpu_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n;
}

int csrc_gpu_plan_create(const csrc_host_matrix* a, const csrc_gpu_strategy* s,
                         csrc_gpu_plan_t* out) {
    return guarded(__func__, [&] {
        if (!out) throw Error("null output");
        *out = nullptr;
        *out = create_plan(a, s, CreateOpts{});
    });
}

int csrc_gpu_plan_create_colored(const csrc_host_matrix* a, const csrc_gpu_strategy* s,
                                 const int32_t* color, int32_t n_colors, csrc_gpu_plan_t* out) {
    return guarded(__func__, [&] {
        if (!out || !color) throw Error("null argument");
        *out = nullptr;
        CreateOpts o;
        o.color = color;
        o.n_colors = n_colors;
        *out = create_plan(a, s, o);
    });
}

int csrc_gpu_plan_create_csr(int32_t n_rows, int32_t n_cols, const int32_t* row_ptr, const int32_t* col_idx,
                             const double* values, const csrc_gpu_strategy* s, csrc_gpu_plan_t* out) {
    return guarded(__func__, [&] {
        if (!out) throw Error("null output");
        *out = nullptr;
        *out = create_csr_plan(n_rows, n_cols, row_ptr, col_idx, values, s);
    });
}

int csrc_gpu_plan_create_rect(const csrc_host_matrix* a, const csrc_gpu_strategy* s, int32_t m_cols,
                              const int32_t* tail_row_ptr, const int32_t* tail_col_idx,
                              const double* tail_values, csrc_gpu_plan_t* out) {
    return guarded(__func__, [&] {
        if (!out) throw Error("null output");
        *out = nullptr;
        CreateOpts o;
        o.m_cols = m_cols;
        o.rect_ptr = tail_row_ptr;
        o.rect_col = tail_col_idx;
        o.rect_val = tail_values;
        if (m_cols == 0) throw Error("ParallelSpmv: rectangular matrix needs m > n (got m=0)");
        *out = create_plan(a, s, o);
    });
}

int csrc_gpu_plan_create_rect_plan(const csrc_host_matrix* a, const csrc_gpu_strategy* s, int32_t m_cols,
                                   const int32_t* tail_row_ptr, const int32_t* tail_col_idx,
                                   const double* tail_values, const int32_t* color, int32_t n_colors,
                                   const int32_t* block_start, int32_t bands, csrc_gpu_plan_t* out) {
    return guarded(__func__, [&] {
        if (!out) throw Error("null output");
        *out = nullptr;
        if ((color != nullptr) == (block_start != nullptr))
            throw Error("rectangular plan: pass exactly one of a colouring or a band partition");
        CreateOpts o;
        o.m_cols = m_cols;
        o.rect_ptr = tail_row_ptr;
        o.rect_col = tail_col_idx;
        o.rect_val = tail_values;
        o.color = color;
        o.n_colors = n_colors;
        o.block_start = block_start;
        o.bands = bands;
        if (m_cols == 0) throw Error("ParallelSpmv: rectangular matrix needs m > n (got m=0)");
        *out = create_plan(a, s, o);
    });
}

int csrc_gpu_plan_get_coloring(csrc_gpu_plan_t plan, int32_t* color, int32_t* n_colors) {
    return guarded(__func__, [&] {
        Plan& P = *checked(plan);
        if (n_colors) *n_colors = P.n_colors;
        if (color && !P.host_color.empty())
            std::memcpy(color, P.host_color.data(), P.host_color.size() * sizeof(int32_t));
    });
}

int csrc_gpu_plan_create_partitioned(const csrc_host_matrix* a, const csrc_gpu_strategy* s,
                                     const int32_t* block_start, int32_t bands,
                                     csrc_gpu_plan_t* out) {
    return guarded(__func__, [&] {
        if (!out || !block_start) throw Error("null argument");
        *out = nullptr;
        CreateOpts o;
        o.block_start = block_start;
        o.bands = bands;
        *out = create_plan(a, s, o);
    });
}

int csrc_gpu_plan_create_band(const csrc_host_matrix* a, const csrc_gpu_strategy* s,
                              int32_t row_begin, int32_t row_end, csrc_gpu_plan_t* out) {
    return guarded(__func__, [&] {
        if (!out) throw Error("null output");
        *out = nullptr;
        CreateOpts o;
        o.band = true;
        o.row_begin = row_begin;
        o.row_end = row_end;
        *out = create_plan(a, s, o);
    });
}

void csrc_gpu_plan_destroy(csrc_gpu_plan_t plan) {
    if (plan) {
        cudaSetDevice(plan->device);
        cudaStreamSynchronize(plan->stream);
        delete plan;
    }
}

int csrc_gpu_plan_get_info(csrc_gpu_plan_t plan, csrc_gpu_plan_info* info) {
    return guarded(__func__, [&] {
        Plan& P = *checked(plan);
        if (!info) throw Error("null info");
        std::memset(info, 0, sizeof(*info));
        info->n = P.n_global;
        info->k = P.k;
        info->kind = P.exec_kind;
        info->dtype = P.dtype;
        info->bands = P.exec_kind == CSRC_KIND_LOCAL_BUFFERS ? P.lb_bands : P.bands;
        info->buffers_allocated = P.exec_kind == CSRC_KIND_LOCAL_BUFFERS ? P.lb_bands : 0;
        info->n_colors = P.n_colors;
        info->row_begin = P.row_begin;
        info->row_end = P.row_end;
        info->lo = P.lo;
        const count_t band_nnz = P.nrows + (P.value_symmetric ? 1 : 2) * P.k;
        info->model_bytes =
            csrc_model_bytes(P.nrows, band_nnz, P.value_symmetric ? 1 : 0, P.dtype);
        size_t dbytes = 0;
        for (const DevBuf* d : {&P.ia, &P.ja, &P.al, &P.au, &P.ad, &P.sched, &P.cta_ptr,
                                &P.band_shift, &P.tile_band, &P.band_rs, &P.spill_shift, &P.buf, &P.boff, &P.blo, &P.bhi, &P.bstart,
                                &P.iv_begin, &P.iv_end, &P.cptr, &P.contrib, &P.rid, &P.cia,
                                &P.cja, &P.cal, &P.cau, &P.cad, &P.cpk, &P.cw_xp, &P.cw_yp, &P.cw_tk, &P.eptr, &P.eidx, &P.eval, &P.eval_t, &P.pbase, &P.pat_off, &P.dx, &P.dy, &P.dxd, &P.dyd, &P.rt_ptr, &P.rt_col, &P.rt_val, &P.sbase, &P.rmeta, &P.sidx, &P.sval, &P.sval_t, &P.xs_tab, &P.xs_clo, &P.xs_chi, &P.xs_cbase})
            if (d->p) dbytes += d->bytes;
        info->device_bytes = static_cast<int64_t>(dbytes);
        info->n_windows = P.exec_kind == CSRC_KIND_WINDOWED || P.exec_kind == CSRC_KIND_LOCAL_BUFFERS
                              ? (P.far_lo <= P.far_hi ? 2 : 1) : 0;
        info->win_lo[0] = 0;
        info->win_hi[0] = P.near_depth;
        info->win_lo[1] = P.far_lo;
        info->win_hi[1] = P.far_hi;
        info->lanes = P.win_lanes;
        info->stages = P.stages;
        info->smem_bytes = static_cast<int32_t>(P.win_smem);
        info->launches_per_apply = P.launches;
        info->captured_fraction = P.captured;
        info->stream_bytes = info->model_bytes;
        info->row_patterns = 0;
        info->x_hi = P.exec_kind == CSRC_KIND_GATHER ? P.x_hi : P.row_end;
        if (P.exec_kind == CSRC_KIND_GATHER) {
            const int64_t ne = P.nrows ? static_cast<int64_t>(2) * P.k : 0;
            const int64_t vs = static_cast<int64_t>(P.vsize());
            // entry values + (indices | per-row pattern start) + eptr + ad, x, y
            info->stream_bytes = ne * vs + (P.gather_pat ? 4 * static_cast<int64_t>(P.nrows) : 4 * ne) +
                                 4 * (static_cast<int64_t>(P.nrows) + 1) + 3 * vs * P.nrows;
            if (P.gather_sell) {
                // padded slice values (+ columns) + rmeta + slice bases + ad, x, y
                const int64_t pe = P.sell_entries;
                const int64_t H = 32 / P.sell_lanes;
                info->stream_bytes = pe * vs + (P.gather_pat ? 0 : 4 * pe) + 4 * static_cast<int64_t>(P.nrows) +
                                     4 * ((static_cast<int64_t>(P.nrows) + H - 1) / H + 1) + 3 * vs * P.nrows;
            }
            info->row_patterns = P.gather_pat ? P.n_patterns : 0;
            info->lanes = P.gather_sell ? P.sell_lanes : P.gather_lanes;
            info->stages = P.gather_buf ? P.gather_nb : 0;
            info->smem_bytes = P.gather_buf ? (P.dtype == CSRC_DTYPE_F64 ? gather_stage_smem<double>(P)
                                                                         : gather_stage_smem<float>(P))
                                            : 0;
        }
        info->gather_form = P.exec_kind != CSRC_KIND_GATHER ? 0 : P.gather_sell ? 3 : P.gather_buf ? 2 : 1;
        info->csr_cols = P.csr_cols;
        if (P.is_csr) {  // CSR model: values + columns + row pointers + x + y
            const int64_t vs = static_cast<int64_t>(P.vsize());
            info->model_bytes = P.k * (vs + 4) + 4 * (static_cast<int64_t>(P.nrows) + 1) +
                                vs * (static_cast<int64_t>(P.csr_cols) + P.nrows);
        }
        info->m_cols = P.m_cols;
        info->rect_nnz = P.rect_nnz;
        if (P.m_cols) {
            // tail: values + columns + row pointers, and the tail part of x (y RMW counted once)
            const int64_t vs = static_cast<int64_t>(P.vsize());
            info->model_bytes += P.rect_nnz * (vs + 4) + 4 * (static_cast<int64_t>(P.nrows) + 1) +
                                 vs * (P.m_cols - P.n_global);
            info->stream_bytes += P.rect_nnz * (vs + 4) + 4 * (static_cast<int64_t>(P.nrows) + 1) +
                                  vs * (P.m_cols - P.n_global) + 2 * vs * P.nrows;
            info->launches_per_apply += 1;
        }
    });
}

int csrc_gpu_spmv(csrc_gpu_plan_t plan, const double* x_host, int64_t x_len, double* y_host) {
    return guarded(__func__, [&] { apply_host(*checked(plan), x_host, x_len, y_host, false); });
}

int csrc_gpu_spmv_transpose(csrc_gpu_plan_t plan, const double* x_host, int64_t x_len,
                            double* y_host) {
    return guarded(__func__, [&] {
        Plan& P = *checked(plan);
        if (P.m_cols) throw Error("spmv_csrc_transpose: rectangular plans have no transpose product");
        if (P.is_csr) throw Error("spmv_csr: CSR plans have no transpose product");
        if (x_len != P.n_global)
            throw Error("spmv_csrc_transpose: x has length " + std::to_string(x_len) +
                        ", expected " + std::to_string(P.n_global));
        apply_host(P, x_host, x_len, y_host, !P.value_symmetric);
    });
}

int csrc_gpu_spmv_device(csrc_gpu_plan_t plan, const void* d_x, void* d_y, void* stream,
                         int32_t flags) {
    return guarded(__func__, [&] {
        Plan& P = *checked(plan);
        cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : P.stream;
        apply_device(P, d_x, d_y, st, (flags & 1) && !P.value_symmetric);
    });
}

int csrc_gpu_spmv_device_graph(csrc_gpu_plan_t plan, const void* d_x, void* d_y, void* stream) {
    return guarded(__func__, [&] {
        Plan& P = *checked(plan);
        cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : P.stream;
        CUDA_OK(cudaSetDevice(P.device));
        if (!P.graph || P.g_x != d_x || P.g_y != d_y || P.g_stream != st) {
            if (P.graph) cudaGraphExecDestroy(P.graph);
            P.graph = nullptr;
            const bool was_timing = P.timing;
            P.timing = false;
            cudaGraph_t g;
            CUDA_OK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
            try {
                apply_device(P, d_x, d_y, st, false);
            } catch (...) {
                cudaStreamEndCapture(st, &g);
                P.timing = was_timing;
                throw;
            }
            CUDA_OK(cudaStreamEndCapture(st, &g));
            P.timing = was_timing;
            CUDA_OK(cudaGraphInstantiate(&P.graph, g, 0));
            cudaGraphDestroy(g);
            P.g_x = d_x;
            P.g_y = d_y;
            P.g_stream = st;
        }
        CUDA_OK(cudaGraphLaunch(P.graph, st));
    });
}

int csrc_gpu_halo_accumulate(csrc_gpu_plan_t plan, void* d_y, int64_t dst_off,
                             const void* d_recv, int64_t len, void* stream) {
    return guarded(__func__, [&] {
        Plan& P = *checked(plan);
        if (len <= 0) return;
        cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : P.stream;
        CUDA_OK(cudaSetDevice(P.device));
        if (P.dtype == CSRC_DTYPE_F64)
            dev::k_halo_add<double><<<grid_for(P.device, len, 256), 256, 0, st>>>(
                static_cast<double*>(d_y) + dst_off, static_cast<const double*>(d_recv), len);
        else
            dev::k_halo_add<float><<<grid_for(P.device, len, 256), 256, 0, st>>>(
                static_cast<float*>(d_y) + dst_off, static_cast<const float*>(d_recv), len);
        CUDA_OK(cudaGetLastError());
    });
}

int csrc_gpu_gather_interior(csrc_gpu_plan_t plan, int32_t* rows_begin, int32_t* rows_end) {
    return guarded(__func__, [&] {
        Plan& P = *checked(plan);
        if (P.exec_kind != CSRC_KIND_GATHER) throw Error("interior rows are defined for gather plans");
        *rows_begin = P.gi0;
        *rows_end = P.gi1;
    });
}

int csrc_gpu_spmv_device_rows(csrc_gpu_plan_t plan, const void* d_x, void* d_y, void* stream, int32_t flags,
                              int32_t rows_begin, int32_t rows_end) {
    return guarded(__func__, [&] {
        Plan& P = *checked(plan);
        if (P.exec_kind != CSRC_KIND_GATHER) throw Error("row-range products need a gather plan");
        if (P.m_cols) throw Error("row-range products need a square plan");
        if (rows_begin < 0 || rows_end > P.nrows || rows_begin > rows_end)
            throw Error("row range [" + std::to_string(rows_begin) + ", " + std::to_string(rows_end) +
                        ") outside the plan's " + std::to_string(P.nrows) + " rows");
        if (rows_begin == rows_end || P.nrows == 0) return;
        if (rows_begin % 256 != 0 || (rows_end % 256 != 0 && rows_end != P.nrows))
            throw Error("row ranges start on a multiple of 256 and end on one or at the last row");
        CUDA_OK(cudaSetDevice(P.device));
        cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : P.stream;
        const bool tr = (flags & 1) != 0 && !P.value_symmetric;
        if (P.dtype == CSRC_DTYPE_F64)
            launch_gather_range<double>(P, tr, static_cast<const double*>(d_x), static_cast<double*>(d_y),
                                        rows_begin, rows_end, st);
        else
            launch_gather_range<float>(P, tr, static_cast<const float*>(d_x), static_cast<float*>(d_y), rows_begin,
                                       rows_end, st);
        CUDA_OK(cudaGetLastError());
    });
}

int csrc_gpu_band_split(csrc_gpu_plan_t plan, int32_t* boundary_rows_end) {
    return guarded(__func__, [&] {
        Plan& P = *checked(plan);
        *boundary_rows_end = P.split;
    });
}

int csrc_gpu_spmv_device_part(csrc_gpu_plan_t plan, const void* d_x, void* d_y, void* stream,
                              int32_t part) {
    return guarded(__func__, [&] {
        Plan& P = *checked(plan);
        if (part != 0 && part != 1) throw Error("part must be 0 (boundary) or 1 (interior)");
        if (P.row_begin == 0 && P.row_end == P.n_global)
            throw Error("partial products need a band plan");
        if (P.exec_kind != CSRC_KIND_WINDOWED)
            throw Error("partial products need the windowed kernel");
        cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : P.stream;
        apply_device(P, d_x, d_y, st, false, part);
    });
}

int csrc_gpu_set_timing(csrc_gpu_plan_t plan, int32_t enabled) {
    return guarded(__func__, [&] { checked(plan)->timing = enabled != 0; });
}

int csrc_gpu_last_timings(csrc_gpu_plan_t plan, csrc_gpu_timings* t) {
    return guarded(__func__, [&] {
        Plan& P = *checked(plan);
        std::memset(t, 0, sizeof(*t));
        if (!P.ev_recorded) return;
        CUDA_OK(cudaEventSynchronize(P.ev[3]));
        float a = 0, b = 0, c = 0;
        CUDA_OK(cudaEventElapsedTime(&a, P.ev[0], P.ev[1]));
        CUDA_OK(cudaEventElapsedTime(&b, P.ev[1], P.ev[2]));
        CUDA_OK(cudaEventElapsedTime(&c, P.ev[2], P.ev[3]));
        t->init_ms = a;
        t->compute_ms = b;
        t->accumulate_ms = c;
    });
}

int csrc_gpu_time_products(csrc_gpu_plan_t plan, const void* d_x, void* d_y, int32_t reps,
                           int64_t flush_bytes, double* ms_out, double* kernel_ms_out) {
    return guarded(__func__, [&] {
        Plan& P = *checked(plan);
        if (reps < 1) throw Error("reps must be >= 1");
        CUDA_OK(cudaSetDevice(P.device));
        if (flush_bytes > 0 && P.flushbuf.bytes < static_cast<size_t>(flush_bytes))
            P.flushbuf.alloc(static_cast<size_t>(flush_bytes));
        const bool was = P.timing;
        P.timing = true;
        cudaStream_t st = P.stream;
        try {
            CUDA_OK(cudaStreamSynchronize(st));
            for (int r = 0; r < reps; ++r) {
                if (flush_bytes > 0)
                    CUDA_OK(cudaMemsetAsync(P.flushbuf.p, r & 0xff, flush_bytes, st));
                apply_device(P, d_x, d_y, st, false);
                float tot = 0, ker = 0;
                CUDA_OK(cudaEventSynchronize(P.ev[3]));
                CUDA_OK(cudaEventElapsedTime(&tot, P.ev[0], P.ev[3]));
                CUDA_OK(cudaEventElapsedTime(&ker, P.ev[1], P.ev[2]));
                ms_out[r] = tot;
                if (kernel_ms_out) kernel_ms_out[r] = ker;
            }
        } catch (...) {
            P.timing = was;
            throw;
        }
        P.timing = was;
    });
}

int csrc_gpu_time_products_host(csrc_gpu_plan_t plan, const double* x_host, int64_t x_len, int32_t reps,
                                int64_t flush_bytes, double* ms_out, double* kernel_ms_out) {
    return guarded(__func__, [&] {
        Plan& P = *checked(plan);
        if (x_len != P.x_len())
            throw Error("ParallelSpmv: x has length " + std::to_string(x_len) + ", expected " +
                        std::to_string(P.x_len()));
        if (P.row_begin != 0 || P.row_end != P.n_global)
            throw Error("host products need a full-matrix plan (use the device entry points for bands)");
        if (P.n_global == 0) return;
        CUDA_OK(cudaSetDevice(P.device));
        const size_t nx = static_cast<size_t>(P.x_len());
        if (!P.dx.p) P.dx.alloc(nx * P.vsize());
        if (!P.dy.p) P.dy.alloc(static_cast<size_t>(P.n_global) * P.vsize());
        if (P.dtype == CSRC_DTYPE_F64) {
            CUDA_OK(cudaMemcpyAsync(P.dx.p, x_host, nx * 8, cudaMemcpyHostToDevice, P.stream));
            CUDA_OK(cudaStreamSynchronize(P.stream));
        } else {
            std::vector<float> xf(x_host, x_host + nx);
            CUDA_OK(cudaMemcpyAsync(P.dx.p, xf.data(), nx * 4, cudaMemcpyHostToDevice, P.stream));
            CUDA_OK(cudaStreamSynchronize(P.stream));
        }
        if (csrc_gpu_time_products(plan, P.dx.p, P.dy.p, reps, flush_bytes, ms_out, kernel_ms_out) != 0)
            throw Error(csrc_gpu_last_error());
    });
}

}  // extern "C"

// One-shot products: spmv_csrc / spmv_csrc_transpose (kernels.hpp:25-65) called
// once on a host matrix, with no plan to amortise. A plan (gather layout,
// windowed schedule) costs seconds of host preprocessing at C5 -- more than the
// reference's own sequential product (0.54 s). Here the CSRC arrays are
// streamed to the device as stored, row chunk by row chunk through two pinned
// staging sets (host memcpy of chunk c+1 overlaps the DMA of chunk c and the
// kernel on chunk c-1), and every chunk runs the global-atomic CSRC kernel
// (k_atomic: no schedule, red.global scatter) into a device y. The host link
// is the bound (4.8 GB at C5); the kernel hides under the copies.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <thread>
#include <vector>

#include "hostlink.cuh"
#include "internal.hpp"
#include "kernels.cuh"

using namespace csrcgpu;

namespace {

#define OS_CUDA(expr)                                                                        \
    do {                                                                                     \
        cudaError_t _e = (expr);                                                             \
        if (_e != cudaSuccess)                                                               \
            throw Error(std::string("CUDA error: ") + cudaGetErrorString(_e) + " at " + #expr); \
    } while (0)

constexpr int64_t kChunkPairs = int64_t(4) << 20;  // pairs per streamed chunk (~80 MB of fp64 CSRC)

// Pinned staging + device buffers, kept per process (per device) so that
// repeated one-shot calls do not pay cudaHostAlloc / cudaMalloc again.
// Staging set b holds one chunk: rebased ia, ja, al, au, and the chunk's rows
// of x and ad (which land at their offsets in the device-resident x / ad).
constexpr int kArrays = 6;  // ia, ja, al, au, x, ad
constexpr size_t kYStage = size_t(32) << 20;

struct OneShotPool {
    int device = -1;
    int64_t rows_cap = 0, n_cap = 0;
    void* h[2][kArrays] = {};
    void* d[2][4] = {};  // ia, ja, al, au per set; x / ad go to dx / dad
    double *dx = nullptr, *dy = nullptr, *dad = nullptr;
    void* hy[2] = {nullptr, nullptr};
    cudaEvent_t copied[2] = {}, done[2] = {}, ydone[2] = {};
    cudaStream_t s_copy = nullptr, s_comp = nullptr;
    std::unique_ptr<CopyPool> pool;
    void ensure(int dev, int64_t rows, int64_t n) {
        if (device != dev || rows > rows_cap) {
            release();
            device = dev;
            rows_cap = std::max<int64_t>(rows, 1 << 20);
            const size_t bytes[kArrays] = {static_cast<size_t>(rows_cap + 1) * 4, static_cast<size_t>(kChunkPairs) * 4,
                                           static_cast<size_t>(kChunkPairs) * 8,  static_cast<size_t>(kChunkPairs) * 8,
                                           static_cast<size_t>(rows_cap) * 8,     static_cast<size_t>(rows_cap) * 8};
            for (int b = 0; b < 2; ++b) {
                for (int k = 0; k < kArrays; ++k) {
                    OS_CUDA(cudaHostAlloc(&h[b][k], bytes[k], cudaHostAllocDefault));
                    if (k < 4) OS_CUDA(cudaMalloc(&d[b][k], bytes[k] + 256));
                }
                OS_CUDA(cudaHostAlloc(&hy[b], kYStage, cudaHostAllocDefault));
                OS_CUDA(cudaEventCreateWithFlags(&copied[b], cudaEventDisableTiming));
                OS_CUDA(cudaEventCreateWithFlags(&done[b], cudaEventDisableTiming));
                OS_CUDA(cudaEventCreateWithFlags(&ydone[b], cudaEventDisableTiming));
            }
            OS_CUDA(cudaStreamCreateWithFlags(&s_copy, cudaStreamNonBlocking));
            OS_CUDA(cudaStreamCreateWithFlags(&s_comp, cudaStreamNonBlocking));
            const int hw = static_cast<int>(std::max(1u, std::thread::hardware_concurrency()));
            pool = std::make_unique<CopyPool>(std::min(hw, 16));
        }
        if (n > n_cap) {
            for (double* q : {dx, dy, dad})
                if (q) cudaFree(q);
            dx = dy = dad = nullptr;
            n_cap = n;
            OS_CUDA(cudaMalloc(&dx, static_cast<size_t>(n) * 8 + 256));
            OS_CUDA(cudaMalloc(&dy, static_cast<size_t>(n) * 8 + 256));
            OS_CUDA(cudaMalloc(&dad, static_cast<size_t>(n) * 8 + 256));
        }
    }
    void release() {
        if (device < 0) return;
        cudaSetDevice(device);
        for (int b = 0; b < 2; ++b) {
            for (int k = 0; k < kArrays; ++k) {
                if (h[b][k]) cudaFreeHost(h[b][k]);
                h[b][k] = nullptr;
            }
            for (int k = 0; k < 4; ++k) {
                if (d[b][k]) cudaFree(d[b][k]);
                d[b][k] = nullptr;
            }
            if (hy[b]) cudaFreeHost(hy[b]);
            hy[b] = nullptr;
            for (cudaEvent_t* e : {&copied[b], &done[b], &ydone[b]}) {
                if (*e) cudaEventDestroy(*e);
                *e = nullptr;
            }
        }
        for (double* q : {dx, dy, dad})
            if (q) cudaFree(q);
        dx = dy = dad = nullptr;
        n_cap = 0;
        if (s_copy) cudaStreamDestroy(s_copy);
        if (s_comp) cudaStreamDestroy(s_comp);
        s_copy = s_comp = nullptr;
        pool.reset();
        device = -1;
    }
};

std::mutex g_pool_mu;
OneShotPool& pool_for() {
    static OneShotPool p;  // process lifetime (released by the driver at exit)
    return p;
}

int lanes_for(int64_t k, int64_t n) {
    const double avg = n ? static_cast<double>(k) / n : 1.0;
    return avg <= 2.5 ? 2 : avg <= 5 ? 4 : avg <= 10 ? 8 : 16;
}

template <int L>
void launch(const int32_t* ia, const int32_t* ja, const double* al, const double* au, const double* ad,
            const double* x, double* y, int32_t nrows, int32_t row0, cudaStream_t st) {
    const int rows_per_block = 256 / L;
    const int64_t blocks = (nrows + rows_per_block - 1) / rows_per_block;
    dev::k_atomic<double, L><<<static_cast<int>(std::min<int64_t>(blocks, 148 * 8)), 256, 0, st>>>(
        ia, ja, al, au, ad, x, y, nrows, row0, 0);
}

struct Trace {
    bool on = std::getenv("CSRC_GPU_ONESHOT_TRACE") != nullptr;
    std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
    void mark(const char* what) {
        if (!on) return;
        const auto now = std::chrono::steady_clock::now();
        std::fprintf(stderr, "oneshot: %-26s %8.2f ms\n", what, std::chrono::duration<double, std::milli>(now - t).count());
        t = now;
    }
};

void run(const MatView& a, const double* xh, double* yh, bool transpose, int device, Trace& tr) {
    OS_CUDA(cudaSetDevice(device));
    std::lock_guard<std::mutex> lk(g_pool_mu);  // one streamed product at a time per process
    const index_t n = a.n;
    // row chunks of <= kChunkPairs pairs (a single longer row gets its own chunk)
    std::vector<index_t> cuts = {0};
    int64_t max_rows = 1;
    for (index_t r = 0; r < n;) {
        index_t e = r + 1;
        while (e < n && static_cast<int64_t>(a.ia[e + 1]) - a.ia[r] <= kChunkPairs) ++e;
        if (static_cast<int64_t>(a.ia[e]) - a.ia[r] > kChunkPairs && e - r > 1) --e;
        cuts.push_back(e);
        max_rows = std::max<int64_t>(max_rows, e - r);
        r = e;
    }
    int64_t max_pairs = 0;
    for (size_t c = 0; c + 1 < cuts.size(); ++c)
        max_pairs = std::max<int64_t>(max_pairs, static_cast<int64_t>(a.ia[cuts[c + 1]]) - a.ia[cuts[c]]);
    if (max_pairs > kChunkPairs) throw Error("spmv_csrc: a row longer than the streaming chunk");
    tr.mark("chunking");
    OneShotPool& P = pool_for();
    P.ensure(device, max_rows, n);
    tr.mark("pool");
    OS_CUDA(cudaMemsetAsync(P.dy, 0, static_cast<size_t>(n) * 8, P.s_comp));
    const double* al = transpose ? a.au : a.al;
    const double* au = transpose ? a.al : a.au;
    const int L = lanes_for(a.k, n);
    const size_t nc = cuts.size() - 1;
    for (size_t c = 0; c < nc; ++c) {
        const int b = static_cast<int>(c & 1);
        const index_t r0 = cuts[c], r1 = cuts[c + 1];
        const int64_t p0 = a.ia[r0], p1 = a.ia[r1];
        if (c >= 2) OS_CUDA(cudaEventSynchronize(P.done[b]));  // kernel c-2 finished with set b
        // stage chunk c: rebased ia, ja, al, au, and rows r0 .. r1 of x and ad (the
        // chunk's lower columns lie below r1: x of earlier chunks is already resident)
        int32_t* hia = static_cast<int32_t*>(P.h[b][0]);
        for (index_t r = r0; r <= r1; ++r) hia[r - r0] = static_cast<int32_t>(a.ia[r] - p0);
        P.pool->copy(P.h[b][1], a.ja + p0, static_cast<size_t>(p1 - p0) * 4);
        P.pool->copy(P.h[b][2], al + p0, static_cast<size_t>(p1 - p0) * 8);
        if (!a.value_symmetric) P.pool->copy(P.h[b][3], au + p0, static_cast<size_t>(p1 - p0) * 8);
        P.pool->copy(P.h[b][4], xh + r0, static_cast<size_t>(r1 - r0) * 8);
        P.pool->copy(P.h[b][5], a.ad + r0, static_cast<size_t>(r1 - r0) * 8);
        auto up = [&](void* dst, const void* src, size_t bytes) {
            if (bytes) OS_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, P.s_copy));
        };
        up(P.d[b][0], P.h[b][0], static_cast<size_t>(r1 - r0 + 1) * 4);
        up(P.d[b][1], P.h[b][1], static_cast<size_t>(p1 - p0) * 4);
        up(P.d[b][2], P.h[b][2], static_cast<size_t>(p1 - p0) * 8);
        if (!a.value_symmetric) up(P.d[b][3], P.h[b][3], static_cast<size_t>(p1 - p0) * 8);
        up(P.dx + r0, P.h[b][4], static_cast<size_t>(r1 - r0) * 8);
        up(P.dad + r0, P.h[b][5], static_cast<size_t>(r1 - r0) * 8);
        OS_CUDA(cudaEventRecord(P.copied[b], P.s_copy));
        OS_CUDA(cudaStreamWaitEvent(P.s_comp, P.copied[b], 0));
        const double* dal = static_cast<const double*>(P.d[b][2]);
        const double* dau = a.value_symmetric ? dal : static_cast<const double*>(P.d[b][3]);
        const int32_t* dia = static_cast<const int32_t*>(P.d[b][0]);
        const int32_t* dja = static_cast<const int32_t*>(P.d[b][1]);
        const int32_t nr = r1 - r0;
        switch (L) {
            case 2: launch<2>(dia, dja, dal, dau, P.dad + r0, P.dx, P.dy, nr, r0, P.s_comp); break;
            case 4: launch<4>(dia, dja, dal, dau, P.dad + r0, P.dx, P.dy, nr, r0, P.s_comp); break;
            case 8: launch<8>(dia, dja, dal, dau, P.dad + r0, P.dx, P.dy, nr, r0, P.s_comp); break;
            default: launch<16>(dia, dja, dal, dau, P.dad + r0, P.dx, P.dy, nr, r0, P.s_comp); break;
        }
        OS_CUDA(cudaGetLastError());
        OS_CUDA(cudaEventRecord(P.done[b], P.s_comp));  // set b free again (its DMA preceded the kernel)
    }
    tr.mark("chunk loop issued");
    // y down through the pool's two pinned buffers: the DMA of part q+1 overlaps
    // the host copy-out of part q
    const size_t ybytes = static_cast<size_t>(n) * 8;
    const size_t parts = (ybytes + kYStage - 1) / kYStage;
    auto issue = [&](size_t q) {
        const size_t off = q * kYStage, len = std::min(kYStage, ybytes - off);
        const int b = static_cast<int>(q & 1);
        OS_CUDA(cudaMemcpyAsync(P.hy[b], reinterpret_cast<const char*>(P.dy) + off, len, cudaMemcpyDeviceToHost,
                                P.s_comp));
        OS_CUDA(cudaEventRecord(P.ydone[b], P.s_comp));
    };
    issue(0);
    for (size_t q = 0; q < parts; ++q) {
        if (q + 1 < parts) issue(q + 1);  // its buffer was drained by the copy-out of part q - 1
        const int b = static_cast<int>(q & 1);
        OS_CUDA(cudaEventSynchronize(P.ydone[b]));
        const size_t off = q * kYStage;
        P.pool->copy(reinterpret_cast<char*>(yh) + off, P.hy[b], std::min(kYStage, ybytes - off));
    }
    tr.mark("chunks done + y down");
}

}  // namespace

extern "C" int csrc_gpu_spmv_oneshot(const csrc_host_matrix* m, const double* x_host, int64_t x_len,
                                     double* y_host, int32_t transpose, int32_t device) {
    return guarded(__func__, [&] {
        Trace tr;
        MatView a = view_of(m, true);
        tr.mark("structure check");
        const char* fn = transpose ? "spmv_csrc_transpose" : "spmv_csrc";
        if (x_len != a.n)
            throw Error(std::string(fn) + ": x has length " + std::to_string(x_len) + ", expected " +
                        std::to_string(a.n));
        if (a.n == 0) return;
        if (!x_host || !y_host) throw Error(std::string(fn) + ": null vector");
        run(a, x_host, y_host, transpose != 0 && !a.value_symmetric, device, tr);
    });
}

// Pageable host <-> device copies at link speed (shared by the plan builder
// and the device CSRC construction).
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <memory>
#include <utility>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "internal.hpp"

namespace csrcgpu {

// Host vectors without value-initialisation: resize() leaves the pages
// untouched, so the multithreaded copy-out below takes the first-touch page
// faults in parallel instead of a serial zero fill.
template <class T>
struct NoInit : std::allocator<T> {
    using value_type = T;
    template <class U>
    struct rebind { using other = NoInit<U>; };
    NoInit() = default;
    template <class U>
    NoInit(const NoInit<U>&) {}
    template <class U, class... A>
    void construct(U* p, A&&... a) {
        if constexpr (sizeof...(A) == 0) {
            ::new (static_cast<void*>(p)) U;
        } else {
            ::new (static_cast<void*>(p)) U(std::forward<A>(a)...);
        }
    }
};
template <class T>
using HVec = std::vector<T, NoInit<T>>;

#define HL_CUDA(expr)                                                                   \
    do {                                                                                \
        cudaError_t _e = (expr);                                                        \
        if (_e != cudaSuccess)                                                          \
            throw Error(std::string("CUDA error: ") + cudaGetErrorString(_e) + " at " + \
                        #expr);                                                         \
    } while (0)

// Pageable host <-> device copies at link speed: two pinned staging buffers;
// the DMA of one chunk overlaps the multithreaded host memcpy of the next.
// (cudaMemcpy from pageable memory ran at 11 GB/s up and 2.7 GB/s down into
// fresh vectors at C5, profiles/r01_assemble_gpu.jsonl.)
inline void pmemcpy(void* dst, const void* src, size_t bytes) {
    const size_t kMinPerThread = size_t(4) << 20;
    const int hw = static_cast<int>(std::max(1u, std::thread::hardware_concurrency()));
    const int t = static_cast<int>(std::min<size_t>(std::min(hw, 16), std::max<size_t>(1, bytes / kMinPerThread)));
    if (t <= 1) {
        std::memcpy(dst, src, bytes);
        return;
    }
    std::vector<std::thread> pool;
    const size_t part = (bytes / t + 63) & ~size_t(63);
    for (int i = 0; i < t; ++i) {
        const size_t o = static_cast<size_t>(i) * part;
        if (o >= bytes) break;
        const size_t len = std::min(part, bytes - o);
        pool.emplace_back([=] { std::memcpy(static_cast<char*>(dst) + o, static_cast<const char*>(src) + o, len); });
    }
    for (auto& th : pool) th.join();
}

class HostLink {
public:
    static constexpr size_t kStage = size_t(64) << 20;
    explicit HostLink(cudaStream_t st) : st_(st) {}
    ~HostLink() {
        for (int b = 0; b < 2; ++b) {
            if (buf_[b]) cudaFreeHost(buf_[b]);
            if (ev_[b]) cudaEventDestroy(ev_[b]);
        }
    }
    HostLink(const HostLink&) = delete;
    HostLink& operator=(const HostLink&) = delete;

    void h2d(void* dev, const void* host, size_t bytes) {
        if (bytes <= kSmall) {
            if (bytes) HL_CUDA(cudaMemcpy(dev, host, bytes, cudaMemcpyHostToDevice));
            return;
        }
        ready();
        size_t c = 0;
        for (size_t off = 0; off < bytes; off += kStage, ++c) {
            const size_t len = std::min(kStage, bytes - off);
            const int b = static_cast<int>(c & 1);
            if (c >= 2) HL_CUDA(cudaEventSynchronize(ev_[b]));  // the DMA that last read buffer b
            pmemcpy(buf_[b], static_cast<const char*>(host) + off, len);
            HL_CUDA(cudaMemcpyAsync(static_cast<char*>(dev) + off, buf_[b], len, cudaMemcpyHostToDevice, st_));
            HL_CUDA(cudaEventRecord(ev_[b], st_));
        }
        HL_CUDA(cudaStreamSynchronize(st_));
    }

    void d2h(void* host, const void* dev, size_t bytes) {
        if (bytes <= kSmall) {
            if (bytes) HL_CUDA(cudaMemcpy(host, dev, bytes, cudaMemcpyDeviceToHost));
            return;
        }
        ready();
        const size_t nc = (bytes + kStage - 1) / kStage;
        auto issue = [&](size_t c) {
            const size_t off = c * kStage, len = std::min(kStage, bytes - off);
            const int b = static_cast<int>(c & 1);
            HL_CUDA(cudaMemcpyAsync(buf_[b], static_cast<const char*>(dev) + off, len, cudaMemcpyDeviceToHost, st_));
            HL_CUDA(cudaEventRecord(ev_[b], st_));
        };
        issue(0);
        for (size_t c = 0; c < nc; ++c) {
            if (c + 1 < nc) issue(c + 1);  // its buffer was drained by the host copy of chunk c - 1
            const int b = static_cast<int>(c & 1);
            HL_CUDA(cudaEventSynchronize(ev_[b]));
            const size_t off = c * kStage;
            pmemcpy(static_cast<char*>(host) + off, buf_[b], std::min(kStage, bytes - off));
        }
    }

private:
    static constexpr size_t kSmall = size_t(8) << 20;
    void ready() {
        for (int b = 0; b < 2; ++b) {
            if (!buf_[b]) HL_CUDA(cudaHostAlloc(&buf_[b], kStage, cudaHostAllocDefault));
            if (!ev_[b]) HL_CUDA(cudaEventCreateWithFlags(&ev_[b], cudaEventDisableTiming));
        }
    }
    cudaStream_t st_;
    void* buf_[2] = {nullptr, nullptr};
    cudaEvent_t ev_[2] = {nullptr, nullptr};
};


}  // namespace csrcgpu

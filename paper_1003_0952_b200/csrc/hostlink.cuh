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
            // on st_ + a sync: a pageable cudaMemcpy may return before its DMA lands, and
            // kernels on non-blocking streams are not ordered after the legacy stream
            if (bytes) {
                HL_CUDA(cudaMemcpyAsync(dev, host, bytes, cudaMemcpyHostToDevice, st_));
                HL_CUDA(cudaStreamSynchronize(st_));
            }
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
            if (bytes) {
                HL_CUDA(cudaMemcpyAsync(host, dev, bytes, cudaMemcpyDeviceToHost, st_));
                HL_CUDA(cudaStreamSynchronize(st_));
            }
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

#include <condition_variable>
#include <mutex>

namespace csrcgpu {

// Persistent fork-join memcpy pool: the host API stages pageable user vectors
// (the reference's std::vector) through pinned buffers chunk by chunk, so the
// copies must be parallel and cheap to start (no thread spawn per chunk).
class CopyPool {
public:
    explicit CopyPool(int threads) : T_(std::max(1, threads)) {
        for (int id = 1; id < T_; ++id) th_.emplace_back([this, id] { worker(id); });
    }
    ~CopyPool() {
        {
            std::lock_guard<std::mutex> g(m_);
            stop_ = true;
            ++gen_;
        }
        cv_.notify_all();
        for (auto& t : th_) t.join();
    }
    CopyPool(const CopyPool&) = delete;
    CopyPool& operator=(const CopyPool&) = delete;

    void copy(void* dst, const void* src, size_t bytes) {
        if (bytes < (size_t(1) << 20) || T_ == 1) {
            std::memcpy(dst, src, bytes);
            return;
        }
        {
            std::lock_guard<std::mutex> g(m_);
            dst_ = static_cast<char*>(dst);
            src_ = static_cast<const char*>(src);
            bytes_ = bytes;
            pending_ = T_ - 1;
            ++gen_;
        }
        cv_.notify_all();
        part(0);
        std::unique_lock<std::mutex> g(m_);
        done_cv_.wait(g, [this] { return pending_ == 0; });
    }

private:
    void part(int id) const {
        const size_t per = (bytes_ / T_ + 63) & ~size_t(63);
        const size_t o = per * static_cast<size_t>(id);
        if (o < bytes_) std::memcpy(dst_ + o, src_ + o, std::min(per, bytes_ - o));
    }
    void worker(int id) {
        uint64_t seen = 0;
        for (;;) {
            {
                std::unique_lock<std::mutex> g(m_);
                cv_.wait(g, [&] { return gen_ != seen; });
                seen = gen_;
                if (stop_) return;
            }
            part(id);
            std::lock_guard<std::mutex> g(m_);
            if (--pending_ == 0) done_cv_.notify_one();
        }
    }
    int T_;
    std::vector<std::thread> th_;
    std::mutex m_;
    std::condition_variable cv_, done_cv_;
    uint64_t gen_ = 0;
    int pending_ = 0;
    bool stop_ = false;
    char* dst_ = nullptr;
    const char* src_ = nullptr;
    size_t bytes_ = 0;
};

inline bool host_pinned(const void* p) {
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return at.type == cudaMemoryTypeHost || at.type == cudaMemoryTypeManaged;
}

}  // namespace csrcgpu

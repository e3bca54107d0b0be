// Colored CSRC kernel, one persistent launch per product: a dependency-driven
// wavefront over (class, block) tasks instead of one full sweep per class.
//
// Reference: colorful_worker (parallel.hpp:399-435) -- zero y, then per
// conflict-free class in ascending order y[i] += ad*x_i + sum al*x_j and
// y[j] += au*x_i with plain read-add-writes, a barrier per class.
//
// Why not one launch per class on the B200: every class touches ~half of x and
// y (a 27-point class's 13 lower neighbours lie in 13 other classes), so C
// classes sweep x and y C times -- 2x the model bytes at C5 in round 1.
//
// Here rows are grouped in blocks of B >= bandwidth consecutive natural rows;
// task (e, b) is class e-1 restricted to block b (e = 0: copy block b of x into
// class-major order and zero its y; e = C+1: copy block b of y back). A row
// writes y only on [i - bw, i], so tasks of different classes more than one
// block apart never write the same y position, and tasks of one class never do
// (the colouring). Task (e, b) therefore only waits for (e-1, b-1 .. b+1); every
// pair of conflicting rows is ordered as in the reference (class order), so the
// result is deterministic and bit-reproducible. CTAs take chunks of tasks from
// a ticket counter in a topological order that keeps all classes of a window
// of ~S + C blocks in flight: x and y of the window stay L2-resident while the
// matrix streams once.
//
// Layout (plan time, capi.cu setup_colored): rows renumbered block-major, then
// class, then ascending -- each task a 32-aligned range of the class-major
// vectors xp / yp, so the x gathers and y updates of consecutive rows are
// consecutive too. Pairs in SELL-32 slices: entry q of row r at
// sbase[r/32] + 32q + r%32 (ja renumbered, al, au); short rows padded with
// (own row, 0, 0), whose scatter is skipped.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace csrcgpu {
namespace dev {


// One chunk: rows [r0, r1) (class-major) of task `task` = e * NB + b; class
// chunks keep their pairs SELL-NT at ebase (entry q of row r0 + t at
// ebase + q NT + t, w entries per row).
struct __align__(16) CwTicket {
    int32_t task, r0, r1, e;
    int64_t ebase;
    int32_t w, pad;
};

template <typename T>
struct ColorWaveArgs {
    const CwTicket* tickets; // in dispatch order
    const int32_t* nch;      // chunks per task
    int32_t* ctr;            // [0] ticket counter, [1 + task] finished chunks (zeroed per product)
    int32_t n_tickets;
    int32_t n_blocks;        // NB
    int32_t n_e;             // C + 2
    int32_t radius;          // R (blocks)
    const int32_t* rid;      // class-major row -> natural row (-1: padding)
    const int32_t* ja;       // class-major column
    const T* al;
    const T* au;
    const T* ad;             // class-major diagonal
    const T* x;              // natural x
    T* y;                    // natural y
    T* xp;                   // class-major x (scratch)
    T* yp;                   // class-major y (scratch)
    int32_t pf_mode;         // chunk prefetch to L2: 0 off, 1 normal, 2 evict_first policy
};

__device__ __forceinline__ uint64_t l2_policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ int ld_acquire(const int32_t* p) {
    int v;
    asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// bulk prefetch of [p, p + bytes) into L2 (16-byte granules; the arrays carry slack)
__device__ __forceinline__ void prefetch_chunk_l2(const void* p, uint32_t bytes, int mode) {
    const uintptr_t a0 = reinterpret_cast<uintptr_t>(p) & ~uintptr_t(15);
    const uint32_t len = (bytes + 31u) & ~15u;
    if (!len || mode == 0) return;
    if (mode == 2) {
        const uint64_t pol = l2_policy_evict_first();
        asm volatile("cp.async.bulk.prefetch.L2.global.L2::cache_hint [%0], %1, %2;" ::"l"(a0), "r"(len), "l"(pol)
                     : "memory");
    } else {
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a0), "r"(len) : "memory");
    }
}

template <typename T>
__device__ __forceinline__ T ld_l2(const T* p) {
    return __ldcg(p);  // y / x scratch written by other SMs in this launch: bypass L1
}

// NT threads per CTA = rows per chunk; U entries per row in flight; MINB
// resident CTAs per SM the register budget targets.
template <typename T, int NT, int U, int MINB>
__global__ void __launch_bounds__(NT, MINB) k_colored_wave(ColorWaveArgs<T> A) {
    __shared__ CwTicket s_tk;
    const int tid = threadIdx.x;
    const int lane = tid & 31;
    // warp 0 owns the dispatch: lane 0 takes tickets (one prefetched ahead, so the
    // counter's round trip overlaps the current chunk) and starts the chunk's matrix
    // data towards L2; lanes 0 .. 2R wait on the dependencies in parallel
    int next = 0;
    if (tid == 0) next = atomicAdd(A.ctr, 1);
    for (;;) {
        if (tid < 32) {
            int task = -1, e = 0;
            if (lane == 0) {
                const int q = next;
                if (q < A.n_tickets) {
                    s_tk = A.tickets[q];
                    task = s_tk.task;
                    e = s_tk.e;
                    next = atomicAdd(A.ctr, 1);  // prefetch; the chunk it names waits its turn
                    if (s_tk.w > 0) {
                        const uint32_t m = static_cast<uint32_t>(s_tk.w) * NT;
                        prefetch_chunk_l2(A.ja + s_tk.ebase, 4u * m, A.pf_mode);
                        prefetch_chunk_l2(A.al + s_tk.ebase, sizeof(T) * m, A.pf_mode);
                        if (A.au != A.al) prefetch_chunk_l2(A.au + s_tk.ebase, sizeof(T) * m, A.pf_mode);
                    }
                } else {
                    s_tk.task = -1;
                }
            }
            task = __shfl_sync(0xffffffffu, task, 0);
            e = __shfl_sync(0xffffffffu, e, 0);
            if (task >= 0 && e >= 1) {
                // (e-1, b-R .. b+R): every earlier task that may share a written y position
                const int b = task % A.n_blocks;
                const int d = b - A.radius + lane;
                if (lane <= 2 * A.radius && d >= 0 && d < A.n_blocks) {
                    const int dep = (e - 1) * A.n_blocks + d;
                    const int need = __ldg(A.nch + dep);
                    while (ld_acquire(A.ctr + 1 + dep) < need) __nanosleep(32);
                }
            }
            __syncwarp();
        }
        __syncthreads();
        const int task = s_tk.task;
        if (task < 0) return;
        const int e = s_tk.e, r0 = s_tk.r0, r1 = s_tk.r1;
        if (e == 0) {
            // x -> class-major xp, zero yp (block b, all classes)
            for (int r = r0 + tid; r < r1; r += NT) {
                const int i = __ldg(A.rid + r);
                __stcg(A.xp + r, i >= 0 ? __ldg(A.x + i) : T(0));
                __stcg(A.yp + r, T(0));
            }
        } else if (e == A.n_e - 1) {
            // class-major yp -> y (block b): final once every class of blocks b .. b+R is done
            for (int r = r0 + tid; r < r1; r += NT) {
                const int i = __ldg(A.rid + r);
                if (i >= 0) A.y[i] = ld_l2(A.yp + r);
            }
        } else {
            // one row per thread: colorful_worker's row update (parallel.hpp:411-434)
            const int r = r0 + tid;
            const int w = s_tk.w;
            const int64_t base = s_tk.ebase + tid;
            if (r < r1) {
                const T xi = ld_l2(A.xp + r);
                T acc = T(0);
                for (int q0 = 0; q0 < w; q0 += U) {
                    int32_t j[U];
                    T vl[U], vu[U], xv[U], yv[U];
#pragma unroll
                    for (int u = 0; u < U; ++u) {
                        const bool in = q0 + u < w;
                        const int64_t ei = base + static_cast<int64_t>(NT) * (q0 + u);
                        j[u] = in ? __ldcs(A.ja + ei) : r;
                        vl[u] = in ? __ldcs(A.al + ei) : T(0);
                        vu[u] = in ? (A.au == A.al ? vl[u] : __ldcs(A.au + ei)) : T(0);
                    }
                    // padding entries (own row) neither gather nor scatter
#pragma unroll
                    for (int u = 0; u < U; ++u) {
                        const bool real = j[u] != r;
                        xv[u] = real ? ld_l2(A.xp + j[u]) : T(0);
                        yv[u] = real ? ld_l2(A.yp + j[u]) : T(0);
                    }
#pragma unroll
                    for (int u = 0; u < U; ++u) {
                        if (j[u] != r) {
                            acc = fma(vl[u], xv[u], acc);
                            __stcg(A.yp + j[u], fma(vu[u], xi, yv[u]));
                        }
                    }
                }
                // y[i] += yi (earlier classes may already have scattered into y[i])
                __stcg(A.yp + r, ld_l2(A.yp + r) + fma(__ldg(A.ad + r), xi, acc));
            }
        }
        __syncthreads();  // every thread's stores of this chunk precede the release below
        if (tid == 0) {
            __threadfence();
            atomicAdd(A.ctr + 1 + task, 1);
        }
    }
}

}  // namespace dev
}  // namespace csrcgpu

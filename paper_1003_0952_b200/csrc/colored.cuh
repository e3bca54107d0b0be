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
    asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p));
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


// ---------------------------------------------------------------------------
// Ring form of the wavefront (the default): the same (class, block) tasks,
// tickets and dependency counters, but every CTA is warp-specialised. A loader
// warp takes tickets ahead of time and streams each chunk's pairs -- packed per
// sub-chunk as [ja | al | au], SELL-128 -- into a shared-memory ring with one
// TMA bulk copy per stage (L2 evict_first: the matrix is read once); a checker
// warp polls the chunk's dependencies while the copy is in flight; four
// consumer warps (one row per thread) wait for the stage and only then touch
// xp / yp in L2; a signaller warp fences and publishes the completion count
// behind them (need = 4 per chunk). The DRAM latency of the matrix stream is
// therefore off the dependency path, and the traffic drops to 1.2-1.3x the model
// (1.65x for the direct form); the x / y window of all classes is
// ~ (C + 2) (bw + rows of the claimed, unfinished tickets) 16 B. There is no
// CTA-wide barrier in the loop. Measured steps and the variants that lost:
// DESIGN.md section 5.4, profiles/r02_colored_ring_sweeps.txt.
constexpr int kCrRows = 128;       // rows per chunk = consumer threads
constexpr int kCrWarps = kCrRows / 32;
constexpr int kCrMaxStages = 6;
constexpr int kCrCopy = 1024;     // positions per copy chunk (tasks e = 0 and e = C + 1)

struct __align__(16) CrHdr {
    int32_t task, r0, r1, e;
    int32_t nq, flags, pad0, pad1;  // flags: 1 first sub-chunk, 2 last
};

template <typename T>
struct ColorRingArgs {
    const CwTicket* tickets;   // ebase = byte offset of the chunk in pk; pad = entries per sub-chunk
    const int32_t* nch;        // chunks per task
    int32_t* ctr;              // [0] ticket counter, [1 + task] finished consumer warps
    int32_t n_tickets, n_blocks, n_e, radius;
    const int32_t* rid;        // class-major row -> natural row (-1: padding)
    const unsigned char* pk;   // packed pairs
    const T* ad;
    const T* x;
    T* y;
    T* xp;
    T* yp;
    int32_t stages, stage_bytes;
    int32_t sym;               // no au section (value-symmetric)
    int32_t tr;                // transpose product: al / au roles swapped
    int32_t pf;                // prefetcher warp on: x / y gather targets of the next chunk warmed in L2
    int32_t claim;             // loader's ticket claim policy (0 eager, 1 after staging, 2 when a stage is free)
};

__device__ __forceinline__ uint64_t l2_policy_evict_last() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}

__device__ __forceinline__ void tma_load_hint(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                              uint64_t pol) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::
            "r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
        : "memory");
}

// xp / yp accesses: L2 only (other SMs write them within the launch); HINT adds an
// evict_last policy so the wavefront window outlives the matrix stream in L2
template <bool HINT>
__device__ __forceinline__ double ld_w(const double* p, uint64_t pol) {
    double v;
    if (HINT)
        asm volatile("ld.global.cg.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
    else
        asm volatile("ld.global.cg.f64 %0, [%1];" : "=d"(v) : "l"(p));
    return v;
}
template <bool HINT>
__device__ __forceinline__ float ld_w(const float* p, uint64_t pol) {
    float v;
    if (HINT)
        asm volatile("ld.global.cg.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(v) : "l"(p), "l"(pol));
    else
        asm volatile("ld.global.cg.f32 %0, [%1];" : "=f"(v) : "l"(p));
    return v;
}
template <bool HINT>
__device__ __forceinline__ void st_w(double* p, double v, uint64_t pol) {
    if (HINT)
        asm volatile("st.global.cg.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(p), "d"(v), "l"(pol));
    else
        asm volatile("st.global.cg.f64 [%0], %1;" ::"l"(p), "d"(v));
}
template <bool HINT>
__device__ __forceinline__ void st_w(float* p, float v, uint64_t pol) {
    if (HINT)
        asm volatile("st.global.cg.L2::cache_hint.f32 [%0], %1, %2;" ::"l"(p), "f"(v), "l"(pol));
    else
        asm volatile("st.global.cg.f32 [%0], %1;" ::"l"(p), "f"(v));
}

__device__ __forceinline__ bool mbar_try(uint64_t* bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n .reg .pred p;\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        " selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}

constexpr int kCrThreads = kCrRows + 128;  // consumers + loader, checker, signaller and prefetcher warps
// SPLIT form: 256 threads (a second warpgroup of the three helper warps + one idle warp)
// and a setmaxnreg register split -- the launch gives every thread 80 registers (3 CTAs per
// SM), the helper warpgroup drops to 40 and the consumers rise to 120, so the U = 14 / 16
// forms (a whole 27-point row's gathers in flight: one L2 round trip per chunk) keep three
// CTAs per SM instead of two.
// (Measured slower, C5 1.58 vs 1.29 ms, and kept opt-in; a 56 / 112 split -- no spills in
// the loader -- did not come up at all: the consumers' setmaxnreg.inc never got its registers.)
constexpr int kCrSplitThreads = 2 * kCrRows;
constexpr int kCrHelperRegs = 40;
constexpr int kCrConsumerRegs = 120;

// Warp roles: consumers 0 .. kCrWarps-1 (one row per thread), loader kCrWarps
// (lane 0: tickets, TMA), checker kCrWarps + 1 (dependency polls ahead of the
// consumers), signaller kCrWarps + 2 (fence + completion count behind them).
// Per stage s:
//   pub[s]   loader -> checker, signaller   the fill's header is written
//   full[s]  loader (TMA bytes) + checker (dependencies met) -> consumers
//   done[s]  consumers + signaller (header read) -> loader (stage free) and
//            signaller (stores issued)
// so a consumer warp's chain per sub-chunk is one L2 round trip: wait full,
// gather x / y, store, arrive done. The poll's round trip runs while the TMA is
// in flight, the fence's while the consumers are on their next chunk.
// LR lanes per row (1 or 2): a chunk holds RC = 128 / LR rows; with two lanes a row's pairs
// are dealt round-robin (lane l takes pairs l, l + 2, ...), thread = row * 2 + lane, so the
// half-batches of a warp's 16 rows are 128-byte segments and the lanes meet in one shuffle.
template <typename T, int U, bool HINT, bool SPLIT, int LR = 1>
__global__ void __launch_bounds__(SPLIT ? kCrSplitThreads : kCrThreads,
                                  SPLIT ? 3 : (LR == 2 ? 4 : (U <= 4 ? 4 : ((U <= 8 || (sizeof(T) == 4 && U <= 14)) ? 3 : 2))))
    k_colored_ring(ColorRingArgs<T> A) {
    static_assert(LR == 1 || LR == 2, "one or two lanes per row");
    constexpr int RC = kCrRows / LR;  // rows per class chunk
    extern __shared__ __align__(128) unsigned char smem_raw[];
    __shared__ __align__(8) uint64_t full[kCrMaxStages];
    __shared__ __align__(8) uint64_t done[kCrMaxStages];
    __shared__ __align__(8) uint64_t pub[kCrMaxStages];
    __shared__ CrHdr hdr[kCrMaxStages];
    const int tid = threadIdx.x;
    const int warp = tid >> 5;
    const int lane = tid & 31;
    const int S = A.stages;
    if (tid == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(&full[s], 2);
            mbar_init(&done[s], kCrWarps + 1 + (A.pf ? 1 : 0));
            mbar_init(&pub[s], 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    if (SPLIT && warp >= kCrWarps) asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kCrHelperRegs));
    if (warp == kCrWarps) {
        // --------------------------------------------------------- loader
        if (lane != 0) return;
        const uint64_t pol = l2_policy_evict_first();
        const int n = A.n_tickets;
        const uint32_t eb = 4u + static_cast<uint32_t>(sizeof(T)) * (A.sym ? 1u : 2u);  // bytes per pair
        // Ticket claims (A.claim): every claimed, unfinished ticket widens the distance the
        // classes must keep (its rows count as in flight), so claiming late keeps the x / y
        // window small; claiming early hides the counter + ticket round trips.
        //   0  two tickets ahead of the one being staged (both round trips hidden)
        //   1  the next ticket once the current one is staged
        //   2  the next ticket only when a stage is free for it
        int idx = atomicAdd(A.ctr, 1);
        int nxt = A.claim == 0 ? atomicAdd(A.ctr, 1) : n;
        bool have = idx < n;
        CwTicket tk{};
        if (have) tk = A.tickets[idx];
        int fill = 0;
        for (;;) {
            bool have_n = false;
            CwTicket tkn{};
            int nn = n;
            if (A.claim == 0) {
                // the next ticket and the index after it are fetched while this one streams
                have_n = nxt < n;
                if (have_n) tkn = A.tickets[nxt];
                nn = have_n ? atomicAdd(A.ctr, 1) : n;
            }
            if (!have) {
                const int s = fill % S;
                mbar_wait(&done[s], ((fill / S) & 1) ^ 1);
                hdr[s].task = -1;
                mbar_arrive(&pub[s]);
                mbar_arrive(&full[s]);
                break;
            }
            const bool cls = tk.e >= 1 && tk.e < A.n_e - 1 && tk.w > 0;
            const int ws = cls ? tk.pad : 1;
            const int nsub = cls ? (tk.w + ws - 1) / ws : 1;
            const unsigned char* src = A.pk + tk.ebase;
            for (int k = 0; k < nsub; ++k, ++fill) {
                const int s = fill % S;
                mbar_wait(&done[s], ((fill / S) & 1) ^ 1);
                const int nq = cls ? min(ws, tk.w - k * ws) : 0;
                CrHdr h;
                h.task = tk.task;
                h.r0 = tk.r0;
                h.r1 = tk.r1;
                h.e = tk.e;
                h.nq = nq;
                h.flags = (k == 0 ? 1 : 0) | (k == nsub - 1 ? 2 : 0);
                h.pad0 = h.pad1 = 0;
                hdr[s] = h;
                mbar_arrive(&pub[s]);
                if (nq) {
                    const uint32_t bytes = static_cast<uint32_t>(nq) * RC * eb;
                    mbar_expect_tx(&full[s], bytes);
                    tma_load_hint(smem_raw + static_cast<size_t>(s) * A.stage_bytes, src, bytes, &full[s], pol);
                    src += bytes;
                } else if (!cls && tk.r1 > tk.r0 && (tk.e == 0 || tk.e == A.n_e - 1)) {
                    // copy chunk: its row ids (32-aligned start, 16-byte granular length; rid is padded)
                    const uint32_t bytes = (static_cast<uint32_t>(tk.r1 - tk.r0) * 4u + 15u) & ~15u;
                    mbar_expect_tx(&full[s], bytes);
                    tma_load_hint(smem_raw + static_cast<size_t>(s) * A.stage_bytes, A.rid + tk.r0, bytes, &full[s], pol);
                } else {
                    mbar_arrive(&full[s]);
                }
            }
            if (A.claim == 0) {
                tk = tkn;
                have = have_n;
                nxt = nn;
            } else {
                if (A.claim == 2) mbar_wait(&done[fill % S], ((fill / S) & 1) ^ 1);  // a stage is free
                idx = atomicAdd(A.ctr, 1);
                have = idx < n;
                if (have) tk = A.tickets[idx];
            }
        }
        return;
    }

    if (warp == kCrWarps + 1) {
        // -------------------------------------------------------- checker
        // polls a chunk's dependencies while its pairs are in flight, then gives full[s]
        // its second arrival. Blocking here only delays this CTA's later fills, which
        // its consumers take in order anyway.
        for (int fc = 0;; ++fc) {
            const int s = fc % S;
            if (lane == 0) mbar_wait(&pub[s], (fc / S) & 1);
            __syncwarp();
            const CrHdr h = hdr[s];
            if (h.task >= 0 && (h.flags & 1) && h.e >= 1) {
                // (e-1, b-R .. b+R): every earlier task that may share a written y position
                const int b = h.task % A.n_blocks;
                const int d = b - A.radius + lane;
                if (lane <= 2 * A.radius && d >= 0 && d < A.n_blocks) {
                    const int dep = (h.e - 1) * A.n_blocks + d;
                    const int need = __ldg(A.nch + dep) * kCrWarps;
                    while (ld_acquire(A.ctr + 1 + dep) < need) __nanosleep(20);
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&full[s]);  // (stop marker: the consumers read it and leave)
            if (h.task < 0) return;
        }
    }

    if (warp == kCrWarps + 2) {
        // ------------------------------------------------------ signaller
        // publishes completion counts behind the consumers, so the fence's round trip is
        // on nobody's critical path. It holds one of done[s]'s arrivals until it has read
        // the fill's header, which keeps the loader from overwriting hdr[s] before that.
        if (lane != 0) return;
        for (int fs = 0;; ++fs) {
            const int s = fs % S;
            mbar_wait(&pub[s], (fs / S) & 1);
            const int task = hdr[s].task;
            const int flags = hdr[s].flags;
            if (task < 0) return;
            mbar_arrive(&done[s]);
            mbar_wait(&done[s], (fs / S) & 1);
            if (flags & 2) {
                __threadfence();  // the consumers' stores (ordered before this thread by done[s]) precede the count
                atomicAdd(A.ctr + 1 + task, kCrWarps);
            }
        }
    }

    if (warp == kCrWarps + 3) {
        // ----------------------------------------------------- prefetcher
        // With a ring of >= 3 stages a chunk is usually released (pairs landed, dependencies
        // met) while the consumers are still on the previous one. This warp walks the
        // chunk's column ids from shared memory and touches the xp / yp lines its rows will
        // gather (prefetch.global.L2: no data returned, no registers held), so the ~13 % of
        // window sectors that fell out of L2 are back before the consumers' single round
        // trip needs them. It holds one of done[s]'s arrivals while it reads the stage.
        if (!A.pf) return;
        for (int fp = 0;; ++fp) {
            const int s = fp % S;
            mbar_wait(&full[s], (fp / S) & 1);
            const CrHdr h = hdr[s];
            if (h.task < 0) return;
            if (h.e >= 1 && h.e < A.n_e - 1 && h.nq > 0) {
                const int32_t* sja = reinterpret_cast<const int32_t*>(smem_raw + static_cast<size_t>(s) * A.stage_bytes);
                const int total = h.nq * RC;
                for (int k = lane; k < total; k += 32) {
                    const int j = sja[k];
                    if (j != h.r0 + (k & (RC - 1))) {
                        asm volatile("prefetch.global.L2 [%0];" ::"l"(A.xp + j));
                        asm volatile("prefetch.global.L2 [%0];" ::"l"(A.yp + j));
                    }
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&done[s]);
        }
    }

    // ----------------------------------------------------------- consumers
    if (SPLIT) asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kCrConsumerRegs));
    const uint64_t pol = HINT ? l2_policy_evict_last() : 0;
    T xi = T(0), acc = T(0), yown = T(0), dr = T(0);
    for (int fill = 0;; ++fill) {
        const int s = fill % S;
        mbar_wait(&full[s], (fill / S) & 1);
        const CrHdr h = hdr[s];
        if (h.task < 0) return;
        const int e = h.e;
        const int r = h.r0 + tid;
        const bool cls = e >= 1 && e < A.n_e - 1;
        if (e == 0) {
            // x -> class-major xp, zero yp (block b, all classes). The loader staged the
            // chunk's row ids with the ring, so the only global round trip is x itself; a
            // copy chunk holds <= kCrCopy positions and every thread's loads go out together
            const int32_t* srid = reinterpret_cast<const int32_t*>(smem_raw + static_cast<size_t>(s) * A.stage_bytes) + tid;
            int32_t i[kCrCopy / kCrRows];
            T v[kCrCopy / kCrRows];
#pragma unroll
            for (int u = 0; u < kCrCopy / kCrRows; ++u) i[u] = r + u * kCrRows < h.r1 ? srid[u * kCrRows] : -1;
#pragma unroll
            for (int u = 0; u < kCrCopy / kCrRows; ++u) v[u] = i[u] >= 0 ? __ldcs(A.x + i[u]) : T(0);  // read once: streaming
#pragma unroll
            for (int u = 0; u < kCrCopy / kCrRows; ++u) {
                const int q = r + u * kCrRows;
                if (q < h.r1) {
                    st_w<HINT>(A.xp + q, v[u], pol);
                    st_w<HINT>(A.yp + q, T(0), pol);
                }
            }
        } else if (!cls) {
            // class-major yp -> y (block b): final once every class of blocks b .. b+R is done
            const int32_t* srid = reinterpret_cast<const int32_t*>(smem_raw + static_cast<size_t>(s) * A.stage_bytes) + tid;
            int32_t i[kCrCopy / kCrRows];
            T v[kCrCopy / kCrRows];
#pragma unroll
            for (int u = 0; u < kCrCopy / kCrRows; ++u) {
                const int q = r + u * kCrRows;
                i[u] = q < h.r1 ? srid[u * kCrRows] : -1;
                v[u] = q < h.r1 ? ld_w<HINT>(A.yp + q, pol) : T(0);
            }
#pragma unroll
            for (int u = 0; u < kCrCopy / kCrRows; ++u)
                if (i[u] >= 0) __stcs(A.y + i[u], v[u]);  // written once: streaming
        } else {
            // LR lanes per row: colorful_worker's row update (parallel.hpp:411-434)
            const int rl = tid / LR, sub = tid % LR;
            const int rc = h.r0 + rl;
            const bool act = rc < h.r1;
            if (h.flags & 1) {
                xi = act ? ld_w<HINT>(A.xp + rc, pol) : T(0);
                // (no other row of this class writes y[rc])
                yown = act && sub == 0 ? ld_w<HINT>(A.yp + rc, pol) : T(0);
                dr = act && sub == 0 ? __ldcs(A.ad + rc) : T(0);
                acc = T(0);
            }
            const int nq = h.nq;
            const unsigned char* st = smem_raw + static_cast<size_t>(s) * A.stage_bytes;
            const int32_t* sja = reinterpret_cast<const int32_t*>(st) + rl;
            const T* sv0 = reinterpret_cast<const T*>(st + static_cast<size_t>(nq) * RC * 4) + rl;
            const T* sv1 = A.sym ? sv0 : sv0 + static_cast<size_t>(nq) * RC;
            const T* sal = A.tr ? sv1 : sv0;
            const T* sau = A.tr ? sv0 : sv1;
            for (int k0 = 0; k0 * LR + sub < nq; k0 += U) {
                int32_t j[U];
                T xv[U], yv[U];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int q = (k0 + u) * LR + sub;
                    j[u] = q < nq ? sja[q * RC] : rc;
                }
                // padding entries (own row) neither gather nor scatter
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const bool real = j[u] != rc;
                    xv[u] = real ? ld_w<HINT>(A.xp + j[u], pol) : T(0);
                    yv[u] = real ? ld_w<HINT>(A.yp + j[u], pol) : T(0);
                }
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    if (j[u] != rc) {
                        const int q = (k0 + u) * LR + sub;
                        acc = fma(sal[q * RC], xv[u], acc);
                        st_w<HINT>(A.yp + j[u], fma(sau[q * RC], xi, yv[u]), pol);
                    }
                }
            }
            if (h.flags & 2) {
                if (LR == 2) acc += __shfl_xor_sync(0xffffffffu, acc, 1);
                if (act && sub == 0) st_w<HINT>(A.yp + rc, yown + fma(dr, xi, acc), pol);
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&done[s]);  // stage free (loader), stores issued (signaller)
    }
}

}  // namespace dev
}  // namespace csrcgpu

// Transposed-gather CSRC product: y_q = ad_q x_q + sum over the row's stored
// lower pairs (al, ja) + sum over the pairs that name q as their column
// (the "upper" entries a_{q,r} = au[t] for t in row r with ja[t] = q).
//
// The plan (capi.cu setup_gather) lays both parts of each row out as ONE
// contiguous entry stream: eptr[q] .. eptr[q+1] holds the lower entries of q
// (ja / al, in CSRC order) followed by its upper entries (ascending r). No
// scatter, no atomics, no memset: each y element is written exactly once
// with a fixed summation order (bit-reproducible).
//
// Three kernel forms (capi.cu setup_gather picks one per plan):
//   k_gather_staged  the default: a row block's value span (and explicit
//                    columns) staged in shared memory by one TMA bulk copy;
//                    row-pattern compression of the columns (PF = 1)
//   k_gather_sell    SELL-sliced layout, one warp per slice, loads in flight
//                    from registers; chosen for long patterned rows (C4)
//   k_gather_rows    plain L-lanes-per-row fallback for rows whose entry
//                    span does not fit a staging buffer (optional TMA L2
//                    prefetch of future spans, off by default: it hurt)
// Measured alternatives that lost are recorded in DESIGN.md §5.
#pragma once

#include <cstdint>

namespace csrcgpu {
namespace dev {

__device__ __forceinline__ void prefetch_l2(const void* p, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

// 16-byte aligned span covering elements [i0, i1) of a
template <typename E>
__device__ __forceinline__ void prefetch_span(const E* a, int64_t i0, int64_t i1) {
    if (i1 <= i0) return;
    const uintptr_t b0 = reinterpret_cast<uintptr_t>(a + i0) & ~uintptr_t(15);
    const uintptr_t b1 = (reinterpret_cast<uintptr_t>(a + i1) + 15) & ~uintptr_t(15);
    prefetch_l2(reinterpret_cast<const void*>(b0), static_cast<uint32_t>(b1 - b0));
}

// Ordered read-only loads: volatile asm keeps the issue order of a batch of
// independent loads (ptxas otherwise interleaves each gather with its FMA and
// keeps only ~2 loads in flight per thread in the pattern form).
__device__ __forceinline__ double ld_nc(const double* p) {
    double v;
    asm volatile("ld.global.nc.f64 %0, [%1];" : "=d"(v) : "l"(p));
    return v;
}
__device__ __forceinline__ float ld_nc(const float* p) {
    float v;
    asm volatile("ld.global.nc.f32 %0, [%1];" : "=f"(v) : "l"(p));
    return v;
}
__device__ __forceinline__ int32_t ld_nc(const int32_t* p) {
    int32_t v;
    asm volatile("ld.global.nc.s32 %0, [%1];" : "=r"(v) : "l"(p));
    return v;
}
__device__ __forceinline__ double ld_cs(const double* p) {
    double v;
    asm volatile("ld.global.cs.f64 %0, [%1];" : "=d"(v) : "l"(p));
    return v;
}
__device__ __forceinline__ float ld_cs(const float* p) {
    float v;
    asm volatile("ld.global.cs.f32 %0, [%1];" : "=f"(v) : "l"(p));
    return v;
}
__device__ __forceinline__ int32_t ld_cs(const int32_t* p) {
    int32_t v;
    asm volatile("ld.global.cs.s32 %0, [%1];" : "=r"(v) : "l"(p));
    return v;
}

// L lanes per row from global memory; rows = rows[0..count) when `rows` is
// given, else row0 .. row0 + count - 1.
template <typename T, int L, int PF>
__global__ void __launch_bounds__(256) k_gather_rows(const int32_t* __restrict__ eptr,
                                                     const int32_t* __restrict__ eidx,
                                                     const T* __restrict__ eval,
                                                     const T* __restrict__ ad,
                                                     const T* __restrict__ x, T* __restrict__ y,
                                                     const int32_t* __restrict__ rows,
                                                     int32_t row0, int32_t count) {
    const int sub = threadIdx.x % L;
    const int per_block = blockDim.x / L;
    const int64_t stride = static_cast<int64_t>(gridDim.x) * per_block;
    if (PF > 0 && rows == nullptr && threadIdx.x == 0) {
        // warm-up: the first PF iterations' spans
        for (int d = 0; d < PF; ++d) {
            const int64_t f0 = static_cast<int64_t>(blockIdx.x) * per_block + d * stride;
            if (f0 >= count) break;
            const int64_t f1 = f0 + per_block < count ? f0 + per_block : count;
            const int32_t e0 = __ldg(eptr + row0 + f0), e1 = __ldg(eptr + row0 + f1);
            prefetch_span(eidx, e0, e1);
            prefetch_span(eval, e0, e1);
        }
    }
    for (int64_t base = static_cast<int64_t>(blockIdx.x) * per_block; base < count; base += stride) {
        if (PF > 0 && rows == nullptr && threadIdx.x == 0) {
            const int64_t f0 = base + PF * stride;
            if (f0 < count) {
                const int64_t f1 = f0 + per_block < count ? f0 + per_block : count;
                const int32_t e0 = __ldg(eptr + row0 + f0), e1 = __ldg(eptr + row0 + f1);
                prefetch_span(eidx, e0, e1);
                prefetch_span(eval, e0, e1);
            }
        }
        const int64_t i = base + threadIdx.x / L;
        const bool act = i < count;
        T s = T(0);
        int32_t r = 0;
        if (act) {
            r = rows ? __ldg(rows + i) : row0 + static_cast<int32_t>(i);
            const int32_t e0 = __ldg(eptr + r), e1 = __ldg(eptr + r + 1);
            T s2 = T(0);
            int32_t e = e0 + sub;
            for (; e + L < e1; e += 2 * L) {
                s = fma(__ldg(eval + e), __ldg(x + __ldg(eidx + e)), s);
                s2 = fma(__ldg(eval + e + L), __ldg(x + __ldg(eidx + e + L)), s2);
            }
            if (e < e1) s = fma(__ldg(eval + e), __ldg(x + __ldg(eidx + e)), s);
            s += s2;
        }
#pragma unroll
        for (int off = L / 2; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off, L);
        if (act && sub == 0) y[r] = ad ? s + __ldg(ad + r) * __ldg(x + r) : s;
    }
}

// Staged form (k_gather_staged): each block walks row blocks of
// R = blockDim.x / L rows (grid-stride); thread 0 stages a row block's spans
// into shared memory with cp.async.bulk copies completing on an mbarrier.
// A lane then issues all U gathers of x for its next U entries back to back,
// so a row costs one global round trip per U entries instead of one per entry.
//   NB = 2: the next row block is copied while the block computes this one;
//   NB = 1: half the shared memory -> more resident blocks, the copy latency
//           hidden by the other blocks on the SM.
//   PAT = false: eidx and eval spans are staged, column = eidx[e];
//   PAT = true : row-pattern form. Mesh matrices repeat a handful of
//           column-offset patterns (27-point stencil: 27, interior plus
//           boundary cases); the plan stores per row the start of its pattern
//           in a small offset table (pbase, int32) instead of a 4-byte column
//           index per entry: column = row + pat_off[pbase[row] + j]. Only the
//           value span is staged; the table (a few KB) stays in L1.
// The per-row entry order is the same in every form, so for equal L and U
// the results are bit-identical.
template <typename T>
struct GStageArgs {
    const int32_t* eptr;
    const int32_t* eidx;     // !PAT
    const int32_t* pbase;    // PAT: pattern start per row
    const int32_t* pat_off;  // PAT
    const T* eval;
    const T* ad;
    const T* x;
    T* y;
    int32_t row0;       // rows [row0, nrows); row0 a multiple of R
    int32_t nrows;
    int32_t idx_bytes;  // per buffer, 16-aligned (0 when PAT)
    int32_t val_bytes;  // per buffer, 16-aligned
    // XS (pattern form with staged x): the plan groups the stencil's column
    // offsets into K clusters [clo_k, chi_k]; a row block [q0, q0 + R) then
    // reads x only on the K windows [q0 + clo_k, q0 + R + chi_k), which thread 0
    // copies next to the values (cluster k at element cbase_k of the x area);
    // xs_tab[pattern entry] = cbase_k + alignment pad + (offset - clo_k), so the
    // x value of entry f of local row rl is x_area[xs_tab[.] + rl] (LDS).
    const int32_t* xs_tab;
    const int32_t* clo;
    const int32_t* chi;
    const int32_t* cbase;
    int32_t n_clusters;
    int32_t x_min, x_max;  // readable x range (kernel coordinates)
    int32_t xs_bytes;      // x area per buffer, 16-aligned
    // Row setup staged with the values (rs_bytes > 0): thread 0's copy also
    // brings the row block's eptr[q0 .. q0 + R] and (PAT) pbase[q0 .. q0 + R),
    // so a row's span is read from shared memory after the barrier wait the
    // block makes anyway, instead of a dependent global load per row block.
    // Measured slower (the extra small copies cost more than the load latency
    // they hide): opt-in, CSRC_GPU_GROWS=1.
    int32_t rs_bytes;      // row-setup area per buffer (0 = global loads)
};

// one int32 row array of a row block of R rows (+1 for eptr, + alignment pad)
__host__ __device__ inline int gather_rows_bytes(int R) { return ((R + 8) * 4 + 15) & ~15; }

// shared-memory bytes of one buffer holding up to `cap` entries (+ alignment slack)
__host__ __device__ inline int gather_idx_bytes(int cap) { return ((cap + 8) * 4 + 15) & ~15; }
template <typename T>
__host__ __device__ inline int gather_val_bytes(int cap) {
    return ((cap + 8) * static_cast<int>(sizeof(T)) + 15) & ~15;
}

template <typename T, int L, int U, int NB, int PF, int MINB>
__global__ void __launch_bounds__(256, MINB) k_gather_staged(const GStageArgs<T> A) {
    static_assert(NB == 1 || NB == 2, "one or two row-block buffers");
    constexpr bool PAT = PF >= 1;  // PF: 0 explicit columns, 1 row patterns, 2 patterns + staged x
    constexpr bool XS = PF == 2;
    extern __shared__ __align__(128) unsigned char smem[];
    const int R = blockDim.x / L;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem);  // [2]
    unsigned char* bufs = smem + 16;
    const int buf_bytes = A.idx_bytes + A.val_bytes + (XS ? A.xs_bytes : 0) + A.rs_bytes;
    const int rs_off = A.idx_bytes + A.val_bytes + (XS ? A.xs_bytes : 0);  // row-setup area in a buffer
    const uint32_t rs_e = static_cast<uint32_t>(gather_rows_bytes(R));
    const int sub = threadIdx.x % L;
    const int rrel = threadIdx.x / L;
    const int64_t stride = static_cast<int64_t>(gridDim.x) * R;
    const int64_t first = A.row0 + static_cast<int64_t>(blockIdx.x) * R;
    // thread 0: entry span of the next row block to stage (register pipeline)
    int32_t nx0 = 0, nx1 = 0;
    auto span = [&](int64_t b, int32_t& e0, int32_t& e1) {
        if (b < A.nrows) {
            e0 = __ldg(A.eptr + b);
            e1 = __ldg(A.eptr + (b + R < A.nrows ? b + R : A.nrows));
        }
    };
    auto issue = [&](int buf, int32_t e0, int32_t e1, int64_t q0) {
        unsigned char* st = bufs + buf * buf_bytes;
        const Seg<T> sv = seg(A.eval, e0, e1);
        if (XS) {
            // value span + the K x windows of row block [q0, q0 + R), clamped to
            // the readable x range (the clamped-off slots are never read)
            unsigned char* xa = st + A.idx_bytes + A.val_bytes;
            uint32_t bytes = sv.bytes;
            for (int k = 0; k < A.n_clusters; ++k) {
                const int64_t s0 = q0 + __ldg(A.clo + k), s1 = q0 + R + __ldg(A.chi + k);
                const int64_t c0 = s0 > A.x_min ? s0 : A.x_min, c1 = s1 < A.x_max ? s1 : A.x_max;
                if (c0 < c1) bytes += seg(A.x, c0, c1).bytes;
            }
            mbar_expect_tx(&full[buf], bytes);
            tma_load(st + A.idx_bytes, sv.src, sv.bytes, &full[buf]);
            for (int k = 0; k < A.n_clusters; ++k) {
                const int64_t s0 = q0 + __ldg(A.clo + k), s1 = q0 + R + __ldg(A.chi + k);
                const int64_t c0 = s0 > A.x_min ? s0 : A.x_min, c1 = s1 < A.x_max ? s1 : A.x_max;
                if (c0 >= c1) continue;
                const Seg<T> sx = seg(A.x, c0, c1);
                const uintptr_t ua = reinterpret_cast<uintptr_t>(A.x + s0) & ~uintptr_t(15);
                tma_load(xa + sizeof(T) * __ldg(A.cbase + k) + (reinterpret_cast<uintptr_t>(sx.src) - ua), sx.src,
                         sx.bytes, &full[buf]);
            }
            return;
        }
        uint32_t rs_tx = 0;
        Seg<int32_t> se{}, sp{};
        if (A.rs_bytes) {
            const int64_t q1 = q0 + R < A.nrows ? q0 + R : A.nrows;
            se = seg(A.eptr, q0, q1 + 1);
            rs_tx = se.bytes;
            if (PAT) {
                sp = seg(A.pbase, q0, q1);
                rs_tx += sp.bytes;
            }
        }
        if (PAT) {
            mbar_expect_tx(&full[buf], sv.bytes + rs_tx);
        } else {
            const Seg<int32_t> si = seg(A.eidx, e0, e1);
            mbar_expect_tx(&full[buf], si.bytes + sv.bytes + rs_tx);
            tma_load(st, si.src, si.bytes, &full[buf]);
        }
        tma_load(st + A.idx_bytes, sv.src, sv.bytes, &full[buf]);
        if (A.rs_bytes) {
            tma_load(st + rs_off, se.src, se.bytes, &full[buf]);
            if (PAT) tma_load(st + rs_off + rs_e, sp.src, sp.bytes, &full[buf]);
        }
    };
    if (threadIdx.x == 0) {
        mbar_init(&full[0], 1);
        mbar_init(&full[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        if (first < A.nrows) {
            int32_t e0 = 0, e1 = 0;
            span(first, e0, e1);
            issue(0, e0, e1, first);
        }
        span(first + stride, nx0, nx1);
    }
    __syncthreads();
    constexpr int kIdxAlign = 4;
    constexpr int kValAlign = 16 / sizeof(T);
    int it = 0;
    for (int64_t base = first; base < A.nrows; base += stride, ++it) {
        const int buf = NB == 2 ? (it & 1) : 0;
        if (NB == 2 && threadIdx.x == 0 && base + stride < A.nrows) {
            issue(buf ^ 1, nx0, nx1, base + stride);  // buffer buf^1 was released by the last __syncthreads
            span(base + 2 * stride, nx0, nx1);
        }
        const int64_t row = base + rrel;
        const bool act = row < A.nrows;
        int32_t eb = 0, ee = 0, pb = 0, e_base = 0;
        T d = T(0), xr = T(0);
        if (act && A.ad) {  // CSR plans carry the diagonal in the entry stream (ad == nullptr)
            d = __ldg(A.ad + row);
            xr = __ldg(A.x + row);
        }
        if (!A.rs_bytes) {
            e_base = __ldg(A.eptr + base);  // the row block's first entry
            if (act) {
                eb = __ldg(A.eptr + row);
                ee = __ldg(A.eptr + row + 1);
                if (PAT) pb = __ldg(A.pbase + row) - eb;  // pattern slot of entry f = pb + f
            }
        }
        mbar_wait(&full[buf], NB == 2 ? ((it >> 1) & 1) : (it & 1));
        const uint32_t st = smem_u32(bufs + buf * buf_bytes);
        if (A.rs_bytes) {
            const uint32_t ra = st + static_cast<uint32_t>(rs_off);
            const uint32_t eo = static_cast<uint32_t>((reinterpret_cast<uintptr_t>(A.eptr + base) & 15) >> 2);
            e_base = lds_i(ra + 4u * eo);
            if (act) {
                eb = lds_i(ra + 4u * (eo + rrel));
                ee = lds_i(ra + 4u * (eo + rrel + 1));
                if (PAT) {
                    const uint32_t po = static_cast<uint32_t>((reinterpret_cast<uintptr_t>(A.pbase + base) & 15) >> 2);
                    pb = lds_i(ra + rs_e + 4u * (po + rrel)) - eb;
                }
            }
        }
        const uint32_t ib = st - 4u * static_cast<uint32_t>(e_base & ~(kIdxAlign - 1));
        const uint32_t vb = st + A.idx_bytes -
                            static_cast<uint32_t>(sizeof(T)) * static_cast<uint32_t>(e_base & ~(kValAlign - 1));
        const uint32_t xb = st + A.idx_bytes + A.val_bytes + static_cast<uint32_t>(sizeof(T)) * rrel;
        const int32_t rq = static_cast<int32_t>(row);  // kernel coordinates fit int32
        T acc0 = T(0), acc1 = T(0);
        for (int32_t e = eb + sub; e < ee; e += U * L) {
            T xv[U];
            if (XS) {
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int32_t f = e + u * L;
                    xv[u] = T(0);
                    if (f < ee) xv[u] = lds_f(xb + static_cast<uint32_t>(sizeof(T)) * __ldg(A.xs_tab + pb + f), T());
                }
            } else {
                // all U column ids, then all U gathers of x: 32-bit ids and one IMAD.WIDE per
                // address (the 64-bit row-pointer form cost 4 integer ops per gather and
                // 11 % at C5 fp32); volatile ordered loads measured the same as __ldg here
                int32_t c[U];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int32_t f = e + u * L;
                    c[u] = rq;
                    if (f < ee) c[u] = PAT ? rq + __ldg(A.pat_off + (pb + f)) : lds_i(ib + 4u * f);
                }
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    xv[u] = T(0);
                    if (e + u * L < ee) xv[u] = __ldg(A.x + c[u]);
                }
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int32_t f = e + u * L;
                if (f < ee) {
                    if (u & 1)
                        acc1 = fma(lds_f(vb + sizeof(T) * f, T()), xv[u], acc1);
                    else
                        acc0 = fma(lds_f(vb + sizeof(T) * f, T()), xv[u], acc0);
                }
            }
        }
        T s = acc0 + acc1;
#pragma unroll
        for (int off = L / 2; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off, L);
        if (act && sub == 0) A.y[row] = A.ad ? s + d * xr : s;
        __syncthreads();
        if (NB == 1 && threadIdx.x == 0 && base + stride < A.nrows) {
            issue(0, nx0, nx1, base + stride);  // single buffer: refill once every thread is done with it
            span(base + 2 * stride, nx0, nx1);
        }
    }
}


// Sliced form (k_gather_sell, the default for mesh matrices): the entry
// stream re-laid out in slices of H = 32 / L consecutive rows, one warp per
// slice, L lanes per row. Entry j of the slice's local row rl sits at
//     sbase[s] + 32 (j / L) + L rl + (j % L)
// (SELL-H with L-way interleave; rows shorter than the slice's longest are
// padded, the padding never read), so every value load of a warp is one
// contiguous 32 x sizeof(T) segment, and in the row-pattern form the x gather
// of step t is one contiguous run too (H consecutive rows, same stencil
// offsets). Each lane issues the U value and U x loads of its next U entries
// back to back from registers: no shared-memory staging, no block barriers,
// no TMA round trip per row block -- bytes in flight per SM are set by
// registers (U x 2 x sizeof(T) per thread), not by a staged buffer held for a
// whole compute phase (k_gather_staged). Values and columns are read once:
// evict-first (ld.global.cs).
//   rmeta[row]: PAT: pattern start | len << 20 (offset table <= 2^14 entries,
//               held in shared memory; len < 2^11); explicit: len, columns in sidx.
// Summation order per row: lane sub takes entries j = sub + L t, even t into
// acc0, odd t into acc1; acc0 + acc1; xor-shuffle over the L lanes; + ad x.
// Identical in both forms and for every launch split (host pipeline chunks).
template <typename T>
struct GSellArgs {
    const int32_t* sbase;    // [n_slices + 1] entry offset of each slice
    const int32_t* rmeta;    // [nrows]
    const int32_t* sidx;     // !PAT: columns, slice layout
    const int32_t* pat_off;  // PAT
    const T* sval;           // values, slice layout
    const T* ad;
    const T* x;
    T* y;
    int32_t slice0, slice1;  // slices [slice0, slice1)
    int32_t nrows;           // rows >= nrows are skipped (last slice)
    int32_t pat_len;         // PAT: table entries copied to shared memory
};

// resident 256-thread blocks per SM the register budget is sized for
template <int U> struct SellMinBlocks { static constexpr int value = U <= 4 ? 4 : U <= 9 ? 3 : 2; };

template <typename T, int L, bool PAT, int U>
__global__ void __launch_bounds__(256, SellMinBlocks<U>::value) k_gather_sell(const GSellArgs<T> A) {
    static_assert(L == 1 || L == 2 || L == 4, "lanes per row");
    constexpr int H = 32 / L;
    // PAT: the offset table (a few KB for mesh stencils) lives in shared memory,
    // so each x gather waits on a ~30-cycle LDS instead of an L1 round trip
    extern __shared__ __align__(16) int32_t s_pat[];
    if (PAT) {
        for (int i = threadIdx.x; i < A.pat_len; i += blockDim.x) s_pat[i] = __ldg(A.pat_off + i);
        __syncthreads();
    }
    const int lane = threadIdx.x & 31;
    const int sub = lane % L;
    const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
    for (int64_t s = A.slice0 + ((static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5);
         s < A.slice1; s += nwarps) {  // warp-uniform: the shuffles below see all 32 lanes
        const int32_t row = static_cast<int32_t>(s * H + lane / L);
        const bool act = row < A.nrows;
        int32_t nt = 0, pb = 0;
        if (act) {
            const int32_t meta = __ldg(A.rmeta + row);
            const int32_t len = PAT ? (meta >> 20) : meta;
            pb = PAT ? (meta & 0xFFFFF) + sub : 0;
            nt = len > sub ? (len - sub + L - 1) / L : 0;  // this lane's entries
        }
        const int64_t base = static_cast<int64_t>(__ldg(A.sbase + s)) + lane;
        const T* vp = A.sval + base;
        const int32_t* ip = A.sidx + base;
        T acc0 = T(0), acc1 = T(0);
        // U steps at a time: U offset/column loads, U value loads, U x gathers,
        // each batch predicated on t < nt, then the FMAs in step order. (The
        // predication also keeps ptxas from pairing each gather with its FMA,
        // which makes the in-order warp stall on every load in turn.)
#pragma unroll 1
        for (int32_t t0 = 0; t0 < nt; t0 += U) {
            T v[U], xv[U];
            int32_t c[U];
#pragma unroll
            for (int u = 0; u < U; ++u)
                if (t0 + u < nt)
                    c[u] = PAT ? row + s_pat[pb + L * (t0 + u)] : ld_cs(ip + 32 * static_cast<int64_t>(t0 + u));
#pragma unroll
            for (int u = 0; u < U; ++u)
                if (t0 + u < nt) v[u] = ld_cs(vp + 32 * static_cast<int64_t>(t0 + u));
#pragma unroll
            for (int u = 0; u < U; ++u)
                if (t0 + u < nt) xv[u] = ld_nc(A.x + c[u]);
#pragma unroll
            for (int u = 0; u < U; ++u) {
                if (t0 + u < nt) {
                    if (u & 1)
                        acc1 = fma(v[u], xv[u], acc1);
                    else
                        acc0 = fma(v[u], xv[u], acc0);
                }
            }
        }
        T sum = acc0 + acc1;
#pragma unroll
        for (int off = L / 2; off > 0; off >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, off, L);
        if (act && sub == 0) A.y[row] = A.ad ? sum + __ldg(A.ad + row) * __ldg(A.x + row) : sum;
    }
}

}  // namespace dev
}  // namespace csrcgpu

// sm_100a kernels for the CSRC product y = A x (reference: spmv_csrc,
// kernels.hpp:25-43). Every kernel streams the CSRC arrays once, coalesced;
// they differ in how the transposed scatter y[ja[t]] += au[t] * x[i] is made
// race-free (parallel.hpp:286-435 re-derived for the GPU):
//
//   k_atomic    global-atomic baseline: every scatter is a red.global.add
//   k_colored   one launch per conflict-free row class, plain read-add-write
//   k_windowed  CTA row bands; scatters land in two shared-memory rings
//               (near: distance <= Dn, far: distance in [Fmin, Fmax]) that
//               slide with the tile and are flushed with coalesced
//               red.global.add; the rest spills straight to red.global
//
// Positions are global row/column ids; vectors x and out are indexed
// q + shift (shift = -lo for the device vectors covering [lo, row_end)).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace csrcgpu {
namespace dev {


template <typename T>
__device__ __forceinline__ T ldg_stream(const T* p) {
    return __ldcs(p);  // evict-first: matrix arrays are touched exactly once
}

template <typename T>
__device__ __forceinline__ void red_add(T* p, T v) {
    atomicAdd(p, v);  // result unused -> RED.E.ADD.{F64,F32}
}

// ----------------------------------------------------------------- atomic
// L lanes per row; lanes stride over the row's pairs (coalesced within the
// row segment); the row sum is a shuffle reduction; both the row result and
// every transposed entry go through red.global.add into a zeroed y.
template <typename T, int L>
__global__ void __launch_bounds__(256) k_atomic(const int32_t* __restrict__ ia,
                                                const int32_t* __restrict__ ja,
                                                const T* __restrict__ al,
                                                const T* __restrict__ au,
                                                const T* __restrict__ ad,
                                                const T* __restrict__ x, T* y, int32_t nrows,
                                                int32_t row_begin, int64_t shift) {
    // trip counts are uniform across the block so the width-L shuffles
    // always see all 32 lanes of the warp
    const int sub = threadIdx.x % L;
    const int rows_per_block = blockDim.x / L;
    for (int64_t base = static_cast<int64_t>(blockIdx.x) * rows_per_block; base < nrows;
         base += static_cast<int64_t>(gridDim.x) * rows_per_block) {
        const int64_t r = base + threadIdx.x / L;
        const bool act = r < nrows;
        T s = T(0), xi = T(0);
        if (act) {
            const int64_t g = row_begin + r;
            xi = __ldg(x + g + shift);
            const int32_t t1 = __ldg(ia + r + 1);
            for (int32_t t = __ldg(ia + r) + sub; t < t1; t += L) {
                const int32_t j = ldg_stream(ja + t);
                const T a_l = ldg_stream(al + t);
                const T a_u = au == al ? a_l : ldg_stream(au + t);
                s += a_l * __ldg(x + j + shift);
                red_add(y + j + shift, a_u * xi);
            }
        }
#pragma unroll
        for (int off = L / 2; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off, L);
        if (act && sub == 0) red_add(y + row_begin + r + shift, s + __ldg(ad + r) * xi);
    }
}

// The transposed-gather kernel (CSRC_KIND_GATHER) lives in gather.cuh.

// ---------------------------------------------------------------- colored
// One class per launch (colorful_worker, parallel.hpp:411-434): rows of a
// class share no written y position, so y[j] += and y[i] += are plain
// read-add-writes. The class's rows are stored class-major (row-id list
// `rid`, row pointers `cia` into class-major ja/al/au), so each launch
// streams a contiguous slab.
template <typename T, int L>
__global__ void __launch_bounds__(256) k_colored(const int32_t* __restrict__ rid,
                                                 const int64_t* __restrict__ cia,
                                                 const int32_t* __restrict__ ja,
                                                 const T* __restrict__ al,
                                                 const T* __restrict__ au,
                                                 const T* __restrict__ ad,
                                                 const T* __restrict__ x, T* y, int64_t c0,
                                                 int64_t c1, int64_t shift) {
    const int sub = threadIdx.x % L;
    const int rows_per_block = blockDim.x / L;
    for (int64_t base = c0 + static_cast<int64_t>(blockIdx.x) * rows_per_block; base < c1;
         base += static_cast<int64_t>(gridDim.x) * rows_per_block) {
        const int64_t r = base + threadIdx.x / L;
        const bool act = r < c1;
        T s = T(0), xi = T(0);
        int64_t g = 0;
        if (act) {
            g = __ldg(rid + r);
            xi = __ldg(x + g + shift);
            const int64_t t1 = __ldg(cia + r + 1);
            for (int64_t t = __ldg(cia + r) + sub; t < t1; t += L) {
                const int32_t j = ldg_stream(ja + t);
                const T a_l = ldg_stream(al + t);
                const T a_u = au == al ? a_l : ldg_stream(au + t);
                s += a_l * __ldg(x + j + shift);
                y[j + shift] += a_u * xi;
            }
        }
#pragma unroll
        for (int off = L / 2; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off, L);
        if (act && sub == 0) y[g + shift] += s + ldg_stream(ad + r) * xi;
    }
}

}  // namespace dev
}  // namespace csrcgpu

#include "windowed.cuh"
#include "gather.cuh"

namespace csrcgpu {
namespace dev {

// ------------------------------------------------------------ small kernels
template <typename Tin, typename Tout>
__global__ void k_convert(const Tin* __restrict__ in, Tout* __restrict__ out, int64_t n) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        out[i] = static_cast<Tout>(in[i]);
}

// Rectangular tail (spmv_csrc_rect, kernels.hpp:84-86; ParallelSpmv
// compute_block parallel.hpp:300-304): y[i] += sum_q tval[q] * x[tcol[q]]
// over the CSR tail of row i, tcol already global (n + local column). L lanes
// per row, shuffle reduction, one plain read-add-write of y[i] per row (the
// square product has completed on the same stream).
template <typename T, int L>
__global__ void __launch_bounds__(256) k_rect_tail(const int32_t* __restrict__ tptr,
                                                   const int32_t* __restrict__ tcol,
                                                   const T* __restrict__ tval,
                                                   const T* __restrict__ x, T* y, int32_t nrows) {
    const int sub = threadIdx.x % L;
    const int rows_per_block = blockDim.x / L;
    for (int64_t base = static_cast<int64_t>(blockIdx.x) * rows_per_block; base < nrows;
         base += static_cast<int64_t>(gridDim.x) * rows_per_block) {
        const int64_t r = base + threadIdx.x / L;
        T s = T(0);
        if (r < nrows) {
            const int32_t q1 = __ldg(tptr + r + 1);
            for (int32_t q = __ldg(tptr + r) + sub; q < q1; q += L)
                s += ldg_stream(tval + q) * __ldg(x + ldg_stream(tcol + q));
        }
#pragma unroll
        for (int off = L / 2; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off, L);
        if (r < nrows && sub == 0 && __ldg(tptr + r + 1) > __ldg(tptr + r)) y[r] += s;
    }
}

template <typename T>
__global__ void k_halo_add(T* y, const T* __restrict__ recv, int64_t len) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < len;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        red_add(y + i, recv[i]);
}

// ------------------------------------------------ local-buffers accumulation
// Private band buffers are stored compactly over each band's effective range
// [blo_b, bhi_b] at buf + boff[b] (parallel.hpp:254-255 keeps p dense n-vectors;
// the GPU keeps only the reachable window, the reference's `effective` idea).
// Coverage of y is described by the interval plan (partition.hpp:113-134).
template <typename T>
struct BufArgs {
    T* buf;
    const int64_t* boff;      // per band
    const int32_t* blo;       // per band effective lo
    const int32_t* bhi;       // per band effective hi
    const int32_t* bstart;    // per band first row (global), p+1 entries
    const int32_t* iv_begin;  // intervals
    const int32_t* iv_end;
    const int32_t* cptr;      // contributors
    const int32_t* contrib;
    int32_t n_iv;
    int32_t p;
    int64_t total;            // buffer elements
};

// all_in_one init (parallel.hpp:317-325): the concatenated storage as one slab
template <typename T>
__global__ void k_init_flat(T* buf, int64_t total) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        buf[i] = T(0);
}

// per_buffer / effective init (parallel.hpp:327-338): one CTA row per buffer
template <typename T>
__global__ void k_init_per_buffer(BufArgs<T> B) {
    for (int b = blockIdx.y; b < B.p; b += gridDim.y) {
        const int64_t len = static_cast<int64_t>(B.bhi[b]) - B.blo[b] + 1;
        T* base = B.buf + B.boff[b];
        for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < len;
             i += static_cast<int64_t>(gridDim.x) * blockDim.x)
            base[i] = T(0);
    }
}

// interval init (parallel.hpp:339-346): per interval, its contributors' slices
template <typename T>
__global__ void k_init_interval(BufArgs<T> B) {
    for (int iv = blockIdx.y; iv < B.n_iv; iv += gridDim.y) {
        const int32_t q0 = B.iv_begin[iv], q1 = B.iv_end[iv];
        for (int32_t c = B.cptr[iv]; c < B.cptr[iv + 1]; ++c) {
            const int bb = B.contrib[c];
            T* base = B.buf + B.boff[bb] - B.blo[bb];
            for (int64_t q = q0 + blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
                 q < q1; q += static_cast<int64_t>(gridDim.x) * blockDim.x)
                base[q] = T(0);
        }
    }
}

template <typename T>
__device__ __forceinline__ int find_interval(const BufArgs<T>& B, int32_t q) {
    int lo = 0, hi = B.n_iv;  // first interval with end > q
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (B.iv_end[mid] <= q) lo = mid + 1; else hi = mid;
    }
    return lo;
}

// all_in_one / per_buffer accumulation (parallel.hpp:360-369): y sliced
// evenly; every buffer covering q contributes in ascending id.
template <typename T>
__global__ void k_accum_sliced(BufArgs<T> B, T* y, int32_t q_begin, int32_t q_end,
                               int64_t shift) {
    for (int64_t q = q_begin + blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
         q < q_end; q += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int iv = find_interval(B, static_cast<int32_t>(q));
        T s = T(0);
        if (iv < B.n_iv && B.iv_begin[iv] <= q) {
            for (int32_t c = B.cptr[iv]; c < B.cptr[iv + 1]; ++c) {
                const int bb = B.contrib[c];
                s += B.buf[B.boff[bb] + (q - B.blo[bb])];
            }
        }
        y[q + shift] = s;
    }
}

// effective accumulation (parallel.hpp:371-382): band b sums, for its own
// rows, the buffers whose range covers q (ascending id).
template <typename T>
__global__ void k_accum_effective(BufArgs<T> B, T* y, int64_t shift) {
    for (int b = blockIdx.y; b < B.p; b += gridDim.y) {
        const int32_t q0 = B.bstart[b], q1 = B.bstart[b + 1];
        for (int64_t q = q0 + blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
             q < q1; q += static_cast<int64_t>(gridDim.x) * blockDim.x) {
            // covering buffers of q, ascending id, from the interval plan
            const int iv = find_interval(B, static_cast<int32_t>(q));
            T s = T(0);
            if (iv < B.n_iv && B.iv_begin[iv] <= q) {
                for (int32_t c = B.cptr[iv]; c < B.cptr[iv + 1]; ++c) {
                    const int bb = B.contrib[c];
                    s += B.buf[B.boff[bb] + (q - B.blo[bb])];
                }
            }
            y[q + shift] = s;
        }
    }
}

// interval accumulation (parallel.hpp:384-394)
template <typename T>
__global__ void k_accum_interval(BufArgs<T> B, T* y, int64_t shift) {
    for (int iv = blockIdx.y; iv < B.n_iv; iv += gridDim.y) {
        const int32_t q0 = B.iv_begin[iv], q1 = B.iv_end[iv];
        const int32_t c0 = B.cptr[iv], c1 = B.cptr[iv + 1];
        for (int64_t q = q0 + blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
             q < q1; q += static_cast<int64_t>(gridDim.x) * blockDim.x) {
            T s = T(0);
            for (int32_t c = c0; c < c1; ++c) {
                const int bb = B.contrib[c];
                s += B.buf[B.boff[bb] + (q - B.blo[bb])];
            }
            y[q + shift] = s;
        }
    }
}

}  // namespace dev
}  // namespace csrcgpu

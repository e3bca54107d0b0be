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
// GPU form of the private buffers (parallel.hpp:240-397). Band b's private
// buffer over its effective range [lo_b, hi_b] (partition.hpp:94-102) splits
// in two: positions at or above the band's first row rs_b are written by band b
// alone (no lower band scatters upward), so that part of the buffer IS y; the
// part below, [lo_b, rs_b), is the band's spill buffer at spill + soff[b]
// (k_windowed routes every scatter below rs_b there). The accumulation then
// reduces, for every position q, y[q] (the owner band, the lowest covering id)
// plus the spills of the higher bands covering q in ascending id -- the
// reference's sum over the buffers covering q (parallel.hpp:360-394), in its
// order. Intervals of build_interval_plan (partition.hpp:113-134) with one
// contributor need no work; the four AccumMethods differ in how the init and
// the reduction are decomposed over CTAs, as the reference's do over threads.
template <typename T>
struct BufArgs {
    T* spill;
    const int64_t* soff;      // per band: start of its spill buffer
    const int32_t* blo;       // per band effective lo
    const int32_t* bstart;    // per band first row (global), p+1 entries
    const int32_t* iv_begin;  // intervals
    const int32_t* iv_end;
    const int32_t* cptr;      // contributors (ascending band id)
    const int32_t* contrib;
    int32_t n_iv;
    int32_t p;
    int64_t total;            // spill elements
};

// all_in_one init (parallel.hpp:317-325): the concatenated spill storage as one slab
template <typename T>
__global__ void k_init_flat(T* buf, int64_t total) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        buf[i] = T(0);
}

// per_buffer / effective init (parallel.hpp:327-338): one CTA row per band buffer
template <typename T>
__global__ void k_init_per_buffer(BufArgs<T> B) {
    for (int b = blockIdx.y; b < B.p; b += gridDim.y) {
        const int64_t len = B.soff[b + 1] - B.soff[b];
        T* base = B.spill + B.soff[b];
        for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < len;
             i += static_cast<int64_t>(gridDim.x) * blockDim.x)
            base[i] = T(0);
    }
}

// interval init (parallel.hpp:339-346): per interval, the spill slices of its
// contributors above the owner
template <typename T>
__global__ void k_init_interval(BufArgs<T> B) {
    for (int iv = blockIdx.y; iv < B.n_iv; iv += gridDim.y) {
        const int32_t q0 = B.iv_begin[iv], q1 = B.iv_end[iv];
        for (int32_t c = B.cptr[iv] + 1; c < B.cptr[iv + 1]; ++c) {
            const int bb = B.contrib[c];
            T* base = B.spill + B.soff[bb] - B.blo[bb];
            for (int64_t q = q0 + blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
                 q < q1; q += static_cast<int64_t>(gridDim.x) * blockDim.x)
                base[q] = T(0);
        }
    }
}

// y[q] += the higher contributors' spills at q, ascending id, q in [q0, q1) of
// interval iv; two positions per thread step (16-byte fp64 / 8-byte fp32 pairs
// where the interval is long enough).
template <typename T>
__device__ __forceinline__ void accum_range(const BufArgs<T>& B, T* y, int iv, int64_t q0, int64_t q1,
                                            int64_t shift, int64_t start, int64_t stride) {
    const int32_t c0 = B.cptr[iv] + 1, c1 = B.cptr[iv + 1];
    if (c1 <= c0) return;  // one contributor: the owner's values are already in y
    for (int64_t q = q0 + start; q < q1; q += stride) {
        T s = y[q + shift];
        for (int32_t c = c0; c < c1; ++c) {
            const int bb = B.contrib[c];
            s += B.spill[B.soff[bb] + (q - B.blo[bb])];
        }
        y[q + shift] = s;
    }
}

// all_in_one / per_buffer accumulation (parallel.hpp:360-369): y sliced into
// even slabs (blockIdx.y), each slab walking the intervals it overlaps.
template <typename T>
__global__ void k_accum_sliced(BufArgs<T> B, T* y, int32_t q_begin, int32_t q_end, int64_t shift) {
    const int64_t len = static_cast<int64_t>(q_end) - q_begin;
    const int64_t s0 = q_begin + len * blockIdx.y / gridDim.y, s1 = q_begin + len * (blockIdx.y + 1) / gridDim.y;
    for (int iv = 0; iv < B.n_iv; ++iv) {
        const int64_t a = max(s0, static_cast<int64_t>(B.iv_begin[iv]));
        const int64_t b = min(s1, static_cast<int64_t>(B.iv_end[iv]));
        if (a < b)
            accum_range(B, y, iv, a, b, shift, blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x,
                        static_cast<int64_t>(gridDim.x) * blockDim.x);
    }
}

// effective accumulation (parallel.hpp:371-382): band b (blockIdx.y) sums, for
// its own rows, the buffers covering them (ascending id).
template <typename T>
__global__ void k_accum_effective(BufArgs<T> B, T* y, int64_t shift) {
    for (int b = blockIdx.y; b < B.p; b += gridDim.y) {
        const int64_t r0 = B.bstart[b], r1 = B.bstart[b + 1];
        for (int iv = 0; iv < B.n_iv; ++iv) {
            const int64_t a = max(r0, static_cast<int64_t>(B.iv_begin[iv]));
            const int64_t e = min(r1, static_cast<int64_t>(B.iv_end[iv]));
            if (a < e)
                accum_range(B, y, iv, a, e, shift, blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x,
                            static_cast<int64_t>(gridDim.x) * blockDim.x);
        }
    }
}

// interval accumulation (parallel.hpp:384-394): intervals over blockIdx.y
template <typename T>
__global__ void k_accum_interval(BufArgs<T> B, T* y, int64_t shift) {
    for (int iv = blockIdx.y; iv < B.n_iv; iv += gridDim.y)
        accum_range(B, y, iv, B.iv_begin[iv], B.iv_end[iv], shift,
                    blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x,
                    static_cast<int64_t>(gridDim.x) * blockDim.x);
}

}  // namespace dev
}  // namespace csrcgpu

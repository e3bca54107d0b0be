// Windowed CSRC kernel (the fast path).
//
// GPU re-derivation of the reference's "local buffers" strategy
// (parallel.hpp:286-397: compute_block into a private buffer, then an
// accumulation pass). A CTA's private buffer is a pair of shared-memory rings
// over y positions; the accumulation into y is a coalesced red.global.add of
// every ring slot that leaves the window.
//
//  * Tiles of <= kTileRows rows are staged by TMA (cp.async.bulk, one mbarrier
//    per stage, `stages` deep) into shared memory: ia, ad, ja, al, au of the
//    tile are each one contiguous bulk copy.
//  * L lanes per row (blockDim = kTileRows * L) walk the row's pairs from
//    shared memory, following spmv_csrc (kernels.hpp:32-41):
//      gather   y_i += al[t] * x[ja[t]]      registers, width-L shuffle
//      scatter  y_j += au[t] * x_i           distance d = i - j:
//               d <= Dn            -> near ring
//               Fmin <= d <= Fmax  -> far ring
//               otherwise          -> red.global.add straight into y
//    Ring updates are shared-memory CAS (sm_100a has no native smem FP add);
//    each lane keeps four independent CAS in flight and walks its row's
//    slots with stride B within a batch, so the slot pairs that neighbouring
//    rows share (d and d+1) never meet inside one batch.
//  * Schedule: CTA b processes sched[cta_ptr[b] .. cta_ptr[b+1]); entries
//    flagged kRunStart begin a run of row-contiguous tiles. Within a run the
//    rings slide: after tile [g0, g1) the positions below g1 - Dn (near) and
//    g1 - Fmax (far) are final and are flushed. Rings hold >= window + 2
//    tiles, so that flush never aliases the next tile's slots and a single
//    __syncthreads per tile suffices. Runs of a few tiles dealt round-robin
//    make all CTAs sweep the matrix as one wavefront (far targets and their
//    x stay L2-resident); one run per CTA = contiguous bands (used for the
//    private band buffers of the local-buffers strategy).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace csrcgpu {
namespace dev {

constexpr int kTileRows = 128;      // rows per tile; CTA = kTileRows * L threads
constexpr int kMaxStages = 8;
constexpr int kRunStart = 1 << 30;  // flag bits in TileDesc::r0 (rows < 2^29)
constexpr int kRunEnd = 1 << 29;
constexpr int kRowMask = kRunEnd - 1;

// One tile of a CTA's schedule: rows [r0, r1) (local), pairs [p0, p1);
// r0 carries kRunStart / kRunEnd.
struct __align__(16) TileDesc {
    int32_t r0, r1, p0, p1;
};

template <typename T>
struct WinArgs {
    const int32_t* ia;          // local rows, rebased to 0
    const int32_t* ja;          // global column ids
    const T* al;
    const T* au;
    const T* ad;                // local rows
    const T* x;                 // x[q + xshift]
    T* out;                     // out[q + shift_b]
    const TileDesc* tiles;      // schedule: CTA b owns tiles[cta_ptr[b] .. cta_ptr[b+1])
    const int32_t* cta_ptr;
    const int64_t* band_shift;  // per-CTA output shift (private buffers); null = shift
    int64_t shift;
    int64_t xshift;
    int32_t row_begin;          // global id of local row 0
    int32_t near_depth;         // Dn
    int32_t far_lo, far_hi;     // [Fmin, Fmax]; far_lo > far_hi disables the far ring
    int32_t ring_near;          // RN (power of two)
    int32_t ring_far;           // RF (power of two)
    int32_t max_tile_pairs;
    int32_t stages;             // TMA pipeline depth
    int32_t stage_bytes;
    int32_t x_lo, x_hi;         // global positions valid in x
    int32_t xn_len, xf_len;     // staged x window capacities (elements)
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n .reg .pred p;\n WAIT_%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

// cp.async.bulk global -> shared (TMA 1-D bulk copy, SASS UBLKCP)
__device__ __forceinline__ void tma_load(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
            "r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

// 16-byte aligned window around elements [i0, i1): the copy starts at the
// aligned address below &a[i0]; `off` = elements of padding before a[i0].
template <typename E>
struct Seg {
    const char* src;
    uint32_t bytes;
    uint32_t off;
};

template <typename E>
__device__ __forceinline__ Seg<E> seg(const E* a, int64_t i0, int64_t i1) {
    const uintptr_t b0 = reinterpret_cast<uintptr_t>(a + i0);
    const uintptr_t b1 = reinterpret_cast<uintptr_t>(a + i1);
    const uintptr_t a0 = b0 & ~uintptr_t(15);
    const uintptr_t a1 = (b1 + 15) & ~uintptr_t(15);
    Seg<E> s;
    s.src = reinterpret_cast<const char*>(a0);
    s.bytes = static_cast<uint32_t>(a1 - a0);
    s.off = static_cast<uint32_t>((b0 - a0) / sizeof(E));
    return s;
}

// Stage layout (bytes, each 16-aligned); a segment of m elements of size E
// needs m + 2*(16/E) slots after 16-byte alignment of both ends:
//   ia[kTileRows+1] | ad[kTileRows] | ja[P] | al[P] | au[P]
template <typename T>
struct StageLayout {
    int o_ia, o_ad, o_ja, o_al, o_au, o_xn, o_xf, bytes;
    __host__ __device__ static int al16(int v) { return (v + 15) & ~15; }
    __host__ __device__ static int seg_bytes(int m, int e) { return al16(e * (m + 2 * (16 / e))); }
    // xn_len / xf_len: elements of the near / far x windows (0 = not staged)
    __host__ __device__ StageLayout(int max_pairs, int xn_len, int xf_len) {
        const int e = static_cast<int>(sizeof(T));
        o_ia = 0;
        o_ad = o_ia + seg_bytes(kTileRows + 1, 4);
        o_ja = o_ad + seg_bytes(kTileRows, e);
        o_al = o_ja + seg_bytes(max_pairs, 4);
        o_au = o_al + seg_bytes(max_pairs, e);
        o_xn = o_au + seg_bytes(max_pairs, e);
        o_xf = o_xn + al16(e * xn_len);
        bytes = o_xf + al16(e * xf_len);
    }
};

// Inward 16-byte alignment of the x window [q0, q1) (global positions, x
// indexed as xb[q]): the TMA copy never reads outside [q0, q1); the staged
// positions are [*w0, *w0 + *wn). Positions outside fall back to LDG.
template <typename T>
__device__ __forceinline__ uint32_t x_window(const T* xb, int32_t q0, int32_t q1, int32_t* w0,
                                             int32_t* wn, const char** src) {
    *w0 = q0;
    *wn = 0;
    *src = nullptr;
    if (q1 <= q0) return 0;
    const uintptr_t a = reinterpret_cast<uintptr_t>(xb + q0);
    const uintptr_t b = reinterpret_cast<uintptr_t>(xb + q1);
    const uintptr_t a2 = (a + 15) & ~uintptr_t(15);
    const uintptr_t b2 = b & ~uintptr_t(15);
    if (b2 <= a2) return 0;
    *w0 = q0 + static_cast<int32_t>((a2 - a) / sizeof(T));
    *wn = static_cast<int32_t>((b2 - a2) / sizeof(T));
    *src = reinterpret_cast<const char*>(a2);
    return static_cast<uint32_t>(b2 - a2);
}

// 32-bit shared-memory address forms (no generic-pointer conversions).
__device__ __forceinline__ double lds_f(uint32_t a, double) {
    double v;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a) : "memory");
    return v;
}
__device__ __forceinline__ float lds_f(uint32_t a, float) {
    float v;
    asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a) : "memory");
    return v;
}
__device__ __forceinline__ double cas_s(uint32_t a, double cmp, double val) {
    unsigned long long r;
    asm volatile("atom.shared.cas.b64 %0, [%1], %2, %3;"
                 : "=l"(r)
                 : "r"(a), "l"(__double_as_longlong(cmp)), "l"(__double_as_longlong(val))
                 : "memory");
    return __longlong_as_double(static_cast<long long>(r));
}
__device__ __forceinline__ float cas_s(uint32_t a, float cmp, float val) {
    unsigned r;
    asm volatile("atom.shared.cas.b32 %0, [%1], %2, %3;"
                 : "=r"(r)
                 : "r"(a), "r"(__float_as_uint(cmp)), "r"(__float_as_uint(val))
                 : "memory");
    return __uint_as_float(r);
}

// Shared-memory CAS of a T, as raw bits.
__device__ __forceinline__ double cas_bits(double* p, double cmp, double val) {
    return __longlong_as_double(static_cast<long long>(
        atomicCAS(reinterpret_cast<unsigned long long*>(p),
                  static_cast<unsigned long long>(__double_as_longlong(cmp)),
                  static_cast<unsigned long long>(__double_as_longlong(val)))));
}
__device__ __forceinline__ float cas_bits(float* p, float cmp, float val) {
    return __int_as_float(atomicCAS(reinterpret_cast<int*>(p), __float_as_int(cmp),
                                    __float_as_int(val)));
}
__device__ __forceinline__ bool same_bits(double a, double b) {
    return __double_as_longlong(a) == __double_as_longlong(b);
}
__device__ __forceinline__ bool same_bits(float a, float b) {
    return __float_as_int(a) == __float_as_int(b);
}

template <typename T, int L>
__global__ void __launch_bounds__(kTileRows * L) k_windowed(WinArgs<T> A) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const StageLayout<T> lay(A.max_tile_pairs, A.xn_len, A.xf_len);
    __shared__ __align__(8) uint64_t bars[kMaxStages];
    __shared__ uint32_t offs[kMaxStages][5];
    __shared__ TileDesc descs[kMaxStages];
    __shared__ int4 xwin[kMaxStages];  // staged x windows: near start, len, far start, len

    T* ringN = reinterpret_cast<T*>(smem_raw + A.stages * A.stage_bytes);
    T* ringF = ringN + A.ring_near;

    constexpr int nthreads = kTileRows * L;
    const int tid = threadIdx.x;
    const int maskN = A.ring_near - 1;
    const int maskF = A.ring_far - 1;
    const bool far_on = A.far_lo <= A.far_hi;
    const int b = blockIdx.x;
    const int64_t shift = A.band_shift ? A.band_shift[b] : A.shift;
    T* __restrict__ out = A.out + shift;  // out indexed by global position
    const bool sym = A.au == A.al;
    const int32_t s0 = A.cta_ptr[b];
    const int32_t t_count = A.cta_ptr[b + 1] - s0;
    if (t_count <= 0) return;

    for (int i = tid; i < A.ring_near + (far_on ? A.ring_far : 0); i += nthreads) ringN[i] = T(0);
    if (tid == 0) {
        for (int s = 0; s < A.stages; ++s) mbar_init(&bars[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    // thread 0 issues tile ti's TMA copies from its descriptor (no dependent
    // global loads on the refill path; the next descriptor is prefetched)
    auto issue = [&](int ti, const TileDesc& d) {
        const int s = ti % A.stages;
        const int32_t r0 = d.r0 & kRowMask, r1 = d.r1;
        unsigned char* st = smem_raw + s * A.stage_bytes;
        const Seg<int32_t> s_ia = seg(A.ia, r0, r1 + 1);
        const Seg<T> s_ad = seg(A.ad, r0, r1);
        const Seg<int32_t> s_ja = seg(A.ja, d.p0, d.p1);
        const Seg<T> s_al = seg(A.al, d.p0, d.p1);
        const Seg<T> s_au = seg(A.au, d.p0, d.p1);
        const uint32_t tx =
            s_ia.bytes + s_ad.bytes + s_ja.bytes + s_al.bytes + (sym ? 0u : s_au.bytes);
        offs[s][0] = s_ia.off;
        offs[s][1] = s_ad.off;
        offs[s][2] = s_ja.off;
        offs[s][3] = s_al.off;
        offs[s][4] = s_au.off;
        descs[s] = d;
        // x windows of the tile's ring targets (and own rows)
        const int32_t g0 = A.row_begin + r0, g1 = A.row_begin + r1;
        const T* xb0 = A.x + A.xshift;
        int32_t n0, nn, f0, fn;
        const char *nsrc, *fsrc;
        uint32_t nb = x_window(xb0, max(g0 - A.near_depth, A.x_lo), min(g1, A.x_hi), &n0, &nn, &nsrc);
        uint32_t fb = 0;
        f0 = 0;
        fn = 0;
        fsrc = nullptr;
        if (A.xf_len > 0)
            fb = x_window(xb0, max(g0 - A.far_hi, A.x_lo), min(g1 - A.far_lo, A.x_hi), &f0, &fn, &fsrc);
        xwin[s] = make_int4(n0, nn, f0, fn);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_expect_tx(&bars[s], tx + nb + fb);
        if (nb) tma_load(st + lay.o_xn, nsrc, nb, &bars[s]);
        if (fb) tma_load(st + lay.o_xf, fsrc, fb, &bars[s]);
        tma_load(st + lay.o_ia, s_ia.src, s_ia.bytes, &bars[s]);
        tma_load(st + lay.o_ad, s_ad.src, s_ad.bytes, &bars[s]);
        tma_load(st + lay.o_ja, s_ja.src, s_ja.bytes, &bars[s]);
        tma_load(st + lay.o_al, s_al.src, s_al.bytes, &bars[s]);
        if (!sym) tma_load(st + lay.o_au, s_au.src, s_au.bytes, &bars[s]);
    };
    const TileDesc* my = A.tiles + s0;
    TileDesc next{};  // thread 0: descriptor of the next tile to issue
    if (tid == 0) {
        for (int ti = 0; ti < A.stages && ti < t_count; ++ti) issue(ti, my[ti]);
        if (A.stages < t_count) next = my[A.stages];
    }

    auto flush = [&](T* ring, int mask, int32_t from, int32_t to) {
        if (from < 0) from = 0;
        for (int32_t q = from + tid; q < to; q += nthreads) {
            T* slot = ring + (q & mask);
            const T v = *slot;
            if (v != T(0)) {
                red_add(out + q, v);
                *slot = T(0);
            }
        }
    };

    const int row = tid / L;
    const int sub = tid % L;
    int32_t near_done = 0, far_done = 0;  // flushed-below marks of the current run
    const int32_t near_depth = A.near_depth, far_lo = A.far_lo;
    // far ring test as one unsigned compare; an empty far window never matches
    const uint32_t far_span = far_on ? static_cast<uint32_t>(A.far_hi - A.far_lo) : 0u;
    const uint32_t ringN_s = smem_u32(ringN);
    const uint32_t ringF_s = far_on ? smem_u32(ringF) : 0u;
    const T* __restrict__ xb = A.x + A.xshift;  // x indexed by global position

    for (int ti = 0; ti < t_count; ++ti) {
        const int s = ti % A.stages;
        mbar_wait(&bars[s], (ti / A.stages) & 1);
        const TileDesc dsc = descs[s];
        const int32_t r0 = dsc.r0 & kRowMask, r1 = dsc.r1;
        const int nr = r1 - r0;
        const int32_t g0 = A.row_begin + r0;
        const int32_t g1 = g0 + nr;
        if (dsc.r0 & kRunStart) {
            near_done = g0 - A.near_depth;
            far_done = g0 - A.far_hi;
        }
        const unsigned char* st = smem_raw + s * A.stage_bytes;
        const int32_t* ia_s = reinterpret_cast<const int32_t*>(st + lay.o_ia) + offs[s][0];
        const T* ad_s = reinterpret_cast<const T*>(st + lay.o_ad) + offs[s][1];
        const int32_t* ja_s = reinterpret_cast<const int32_t*>(st + lay.o_ja) + offs[s][2];
        const T* al_s = reinterpret_cast<const T*>(st + lay.o_al) + offs[s][3];
        const T* au_s = sym ? al_s : reinterpret_cast<const T*>(st + lay.o_au) + offs[s][4];
        const int32_t p0 = ia_s[0];
        const int4 xw = xwin[s];
        const T* xn_s = reinterpret_cast<const T*>(st + lay.o_xn);
        const T* xf_s = reinterpret_cast<const T*>(st + lay.o_xf);
        auto xget = [&](int32_t q) -> T {  // staged x, else L1/L2
            if (static_cast<uint32_t>(q - xw.x) < static_cast<uint32_t>(xw.y)) return xn_s[q - xw.x];
            if (static_cast<uint32_t>(q - xw.z) < static_cast<uint32_t>(xw.w)) return xf_s[q - xw.z];
            return __ldg(xb + q);
        };

        const bool act = row < nr;
        const int32_t g = g0 + row;
        T yi = T(0), xi = T(0);
        if (act) {
            xi = xget(g);
            const int32_t a0 = ia_s[row] - p0 + sub;
            const int32_t a1 = ia_s[row + 1] - p0;
            const int32_t m = a0 < a1 ? (a1 - a0 + L - 1) / L : 0;  // pairs of this lane
            const int32_t nb = (m + 3) >> 2;                       // batches; stride nb
            for (int32_t bt = 0; bt < nb; ++bt) {
                int32_t t[4], j[4];
                bool ok[4];
                T xv[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int32_t mm = bt + u * nb;
                    ok[u] = mm < m;
                    t[u] = a0 + mm * L;
                    j[u] = ok[u] ? ja_s[t[u]] : g;
                }
#pragma unroll
                for (int u = 0; u < 4; ++u) xv[u] = ok[u] ? xget(j[u]) : T(0);
                // ring slot (shared address) per pair; 0 = spill / none
                uint32_t sa[4];
                T val[4], old[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const T alv = ok[u] ? al_s[t[u]] : T(0);
                    const T auv = ok[u] ? au_s[t[u]] : T(0);
                    yi += alv * xv[u];
                    val[u] = auv * xi;
                    const int32_t d = g - j[u];
                    const bool nearw = d <= near_depth;
                    const bool farw = static_cast<uint32_t>(d - far_lo) <= far_span;
                    sa[u] = !ok[u] ? 0u
                            : nearw ? ringN_s + (static_cast<uint32_t>(j[u] & maskN) * sizeof(T))
                            : farw  ? ringF_s + (static_cast<uint32_t>(j[u] & maskF) * sizeof(T))
                                    : 0u;
                    if (ok[u] && !nearw && !farw) red_add(out + j[u], val[u]);
                }
                // four independent CAS in flight; retry only on a lost race
#pragma unroll
                for (int u = 0; u < 4; ++u)
                    if (sa[u]) old[u] = lds_f(sa[u], T(0));
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    if (!sa[u]) continue;
                    T seen = cas_s(sa[u], old[u], old[u] + val[u]);
                    while (!same_bits(seen, old[u])) {
                        old[u] = seen;
                        seen = cas_s(sa[u], old[u], old[u] + val[u]);
                    }
                }
            }
        }
        // all 32 lanes reach the width-L reduction (rows >= nr contribute 0)
#pragma unroll
        for (int off = L / 2; off > 0; off >>= 1) yi += __shfl_xor_sync(0xffffffffu, yi, off, L);
        if (act && sub == 0) atomicAdd(ringN + (g & maskN), yi + ad_s[row] * xi);

        __syncthreads();  // stage s consumed; the tile's ring contributions complete
        if (tid == 0 && ti + A.stages < t_count) {
            issue(ti + A.stages, next);
            if (ti + A.stages + 1 < t_count) next = my[ti + A.stages + 1];
        }
        const bool run_ends = (dsc.r0 & kRunEnd) != 0;
        if (run_ends) {
            flush(ringN, maskN, near_done, g1);
            if (far_on) flush(ringF, maskF, far_done, g1 - A.far_lo);
            __syncthreads();  // the next run's window may alias these slots
        } else {
            // slide: positions no later row of the run can reach are final;
            // rings hold window + 2 tiles, so the next tile never aliases them
            flush(ringN, maskN, near_done, g1 - A.near_depth);
            near_done = g1 - A.near_depth;
            if (far_on) {
                flush(ringF, maskF, far_done, g1 - A.far_hi);
                far_done = g1 - A.far_hi;
            }
        }
    }
}

}  // namespace dev
}  // namespace csrcgpu

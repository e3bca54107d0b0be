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
//    shared memory (consumer warps; one extra producer warp issues the TMA
//    copies and flushes the rings), following spmv_csrc (kernels.hpp:32-41):
//      gather   y_i += al[t] * x[ja[t]]      registers, width-L shuffle
//      scatter  y_j += au[t] * x_i           distance d = i - j:
//               d <= Dn            -> near ring
//               Fmin <= d <= Fmax  -> far ring
//               otherwise          -> red.global.add straight into y
//    Ring updates are shared-memory CAS (sm_100a has no native smem FP add);
//    each lane keeps four independent CAS in flight and walks its row's
//    slots with stride B within a batch, so the slot pairs that neighbouring
//    rows share (d and d+1) never meet inside one batch.
//  * Warp specialisation, no __syncthreads in the loop: per stage a "full"
//    mbarrier (TMA complete_tx) and an "empty" mbarrier (one arrival per
//    consumer warp). The producer warp waits for tile ti to be consumed,
//    flushes the ring positions that became final, then refills the stage
//    with tile ti + stages. Consumers never wait on each other.
//  * Schedule: CTA b processes tiles[cta_ptr[b] .. cta_ptr[b+1]); tiles
//    flagged kRunStart begin a run of row-contiguous tiles. Within a run the
//    rings slide: after tile [g0, g1) the positions below g1 - Dn (near) and
//    g1 - Fmax (far) are final. Rings hold window + stages*tile rows so the
//    lagged flush never aliases slots of tiles still in flight; consecutive
//    runs use alternating ring banks (run length >= stages), so a run's
//    final flush overlaps the next run. Runs of a few tiles dealt round-robin
//    make all CTAs sweep the matrix as one wavefront (far targets and their
//    x stay L2-resident); one run per CTA = contiguous bands (used for the
//    private band buffers of the local-buffers strategy).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace csrcgpu {
namespace dev {

constexpr int kTileRows = 128;      // max rows per tile (TR = 32/64/128); CTA = 32 + TR * L threads
constexpr int kMaxStages = 8;
constexpr int kRunStart = 1 << 30;  // flag bits in TileDesc::r0 (rows < 2^29)
constexpr int kRunEnd = 1 << 29;
constexpr int kBank = 1 << 28;      // ring bank of the tile's run
constexpr int kRowMask = kBank - 1;

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
    // local buffers (parallel.hpp:286-397, GPU form): each scheduled tile belongs to one
    // band b; a scatter to q < band_rs[b] (below the band's first row) is band b's
    // out-of-band contribution and goes to its spill buffer spill[q + spill_shift[b]];
    // everything at or above band_rs[b] is band b's alone and goes to out. Null: all to out.
    const int32_t* tile_band;
    const int32_t* band_rs;
    const int64_t* spill_shift;
    T* spill;
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
    int32_t rotate;             // batch-order rotation period (0/1: none)
    int32_t combine;            // ring-free: combine equal-target scatters within a warp
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
    int o_ia, o_ad, o_ja, o_al, o_au, o_xn, o_xf, bytes;  // o_xn/o_xf: optional x windows
    __host__ __device__ static int al16(int v) { return (v + 15) & ~15; }
    __host__ __device__ static int seg_bytes(int m, int e) { return al16(e * (m + 2 * (16 / e))); }
    // xn_len / xf_len: elements of the near / far x windows (0 = not staged)
    __host__ __device__ StageLayout(int max_pairs, int xn_len, int xf_len, int tile_rows = kTileRows) {
        const int e = static_cast<int>(sizeof(T));
        o_ia = 0;
        o_ad = o_ia + seg_bytes(tile_rows + 1, 4);
        o_ja = o_ad + seg_bytes(tile_rows, e);
        o_al = o_ja + seg_bytes(max_pairs, 4);
        o_au = o_al + seg_bytes(max_pairs, e);
        o_xn = o_au + seg_bytes(max_pairs, e);
        o_xf = o_xn + al16(e * xn_len);
        bytes = o_xf + al16(e * xf_len);
    }
};

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

__device__ __forceinline__ int32_t lds_i(uint32_t a) {
    int32_t v;
    asm volatile("ld.shared.s32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
    return v;
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

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

constexpr int kDoneSlots = kMaxStages + 2;  // per-tile "done" barriers (ring)

// Final positions of tile d (stateless: tiles of a run are row-contiguous):
// near [g0 - Dn, g1 - Dn) and far [g0 - Fmax, g1 - Fmax) while the run goes
// on; at the run's end everything the run can still hold.
template <typename T>
__device__ __forceinline__ void flush_tile(const WinArgs<T>& A, T* __restrict__ out, T* rings,
                                           int bank_elems, const TileDesc& d, int lane) {
    const bool far_on = A.far_lo <= A.far_hi;
    const int32_t g0 = A.row_begin + (d.r0 & kRowMask);
    const int32_t g1 = A.row_begin + d.r1;
    T* ringN = rings + ((d.r0 & kBank) ? bank_elems : 0);
    T* ringF = ringN + A.ring_near;
    const bool end = (d.r0 & kRunEnd) != 0;
    auto flush = [&](T* ring, int mask, int32_t from, int32_t to) {
        if (from < 0) from = 0;
        for (int32_t q = from + lane; q < to; q += 32) {
            T* slot = ring + (q & mask);
            const T v = *slot;
            if (v != T(0)) {
                red_add(out + q, v);
                *slot = T(0);
            }
        }
    };
    flush(ringN, A.ring_near - 1, g0 - A.near_depth, end ? g1 : g1 - A.near_depth);
    if (far_on) flush(ringF, A.ring_far - 1, g0 - A.far_hi, end ? g1 - A.far_lo : g1 - A.far_hi);
}

// RINGS = false (the default, capi.cu win_rings): no shared-memory windows --
// every scatter and every row result is a red.global.add; no ring zeroing, no
// done barriers, no flush.
template <typename T, int L, int TR, bool RINGS>
__global__ void __launch_bounds__(32 + TR * L) k_windowed(WinArgs<T> A) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const StageLayout<T> lay(A.max_tile_pairs, 0, 0, TR);
    __shared__ __align__(8) uint64_t full[kMaxStages];
    __shared__ __align__(8) uint64_t empty[kMaxStages];
    __shared__ __align__(8) uint64_t done[kDoneSlots];
    __shared__ uint32_t offs[kMaxStages][5];
    __shared__ TileDesc descs[kMaxStages];
    __shared__ TileDesc dring[kDoneSlots];  // descriptors of recent tiles, for the flush

    constexpr int kConsumerWarps = TR * L / 32;
    const int tid = threadIdx.x;
    const int warp = tid >> 5;
    const int lane = tid & 31;
    const int maskN = A.ring_near - 1;
    const int maskF = A.ring_far - 1;
    const bool far_on = A.far_lo <= A.far_hi;
    const int b = blockIdx.x;
    T* __restrict__ out = A.out + A.shift;  // out indexed by global position
    const bool sym = A.au == A.al;
    const int32_t s0 = A.cta_ptr[b];
    const int32_t t_count = A.cta_ptr[b + 1] - s0;
    if (t_count <= 0) return;
    const int S = A.stages;
    const int bank_elems = A.ring_near + A.ring_far;
    T* rings = reinterpret_cast<T*>(smem_raw + S * A.stage_bytes);

    if (RINGS)
        for (int i = tid; i < 2 * bank_elems; i += blockDim.x) rings[i] = T(0);
    if (tid == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], kConsumerWarps);
        }
        for (int s = 0; s < kDoneSlots; ++s) mbar_init(&done[s], kConsumerWarps);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const TileDesc* my = A.tiles + s0;

    if (warp == 0) {
        // ------------------------------------------------------- producer
        if (lane != 0) return;
        auto issue = [&](int ti, const TileDesc& d) {
            const int s = ti % S;
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
            dring[ti % kDoneSlots] = d;
            // no proxy fence: the empty-barrier wait orders the consumers'
            // reads of this stage before the TMA overwrite (standard pipeline)
            mbar_expect_tx(&full[s], tx);
            tma_load(st + lay.o_ia, s_ia.src, s_ia.bytes, &full[s]);
            tma_load(st + lay.o_ad, s_ad.src, s_ad.bytes, &full[s]);
            tma_load(st + lay.o_ja, s_ja.src, s_ja.bytes, &full[s]);
            tma_load(st + lay.o_al, s_al.src, s_al.bytes, &full[s]);
            if (!sym) tma_load(st + lay.o_au, s_au.src, s_au.bytes, &full[s]);
        };
        for (int ti = 0; ti < S && ti < t_count; ++ti) issue(ti, my[ti]);
        TileDesc next = S < t_count ? my[S] : TileDesc{};
        for (int ti = S; ti < t_count; ++ti) {
            const int s = ti % S;
            mbar_wait(&empty[s], ((ti - S) / S) & 1);  // every consumer is done with tile ti - S
            issue(ti, next);
            if (ti + 1 < t_count) next = my[ti + 1];
        }
        return;
    }

    // --------------------------------------------------------------- consumers
    const int cw = warp - 1;  // consumer warp id
    const int ctid = tid - 32;
    const int row = ctid / L;
    const int sub = ctid % L;
    const int32_t near_depth = A.near_depth, far_lo = A.far_lo;
    const uint32_t far_span = far_on ? static_cast<uint32_t>(A.far_hi - A.far_lo) : 0u;
    const T* __restrict__ xb = A.x + A.xshift;  // x indexed by global position
    for (int ti = 0; ti < t_count; ++ti) {
        const int s = ti % S;
        // lagged flush: tile ti-1 is flushed by consumer warp (ti-1) % W once
        // every consumer warp has finished it
        if (RINGS && ti >= 1 && (ti - 1) % kConsumerWarps == cw) {
            mbar_wait(&done[(ti - 1) % kDoneSlots], ((ti - 1) / kDoneSlots) & 1);
            flush_tile(A, out, rings, bank_elems, dring[(ti - 1) % kDoneSlots], lane);
            __syncwarp();
        }
        mbar_wait(&full[s], (ti / S) & 1);
        const TileDesc dsc = descs[s];
        int32_t rs = INT32_MIN;  // scatters below rs go to the tile's band spill buffer
        T* sp = out;
        if (!RINGS && A.tile_band) {
            const int32_t bnd = A.tile_band[s0 + ti];
            rs = A.band_rs[bnd];
            sp = A.spill + A.spill_shift[bnd];
        }
        const int32_t r0 = dsc.r0 & kRowMask;
        const int nr = dsc.r1 - r0;
        const int32_t g0 = A.row_begin + r0;
        const uint32_t ringN_s = smem_u32(rings + ((dsc.r0 & kBank) ? bank_elems : 0));
        const uint32_t ringF_s = ringN_s + A.ring_near * sizeof(T);
        // 32-bit shared addresses of the staged segments (no generic pointers)
        const uint32_t st_s = smem_u32(smem_raw) + s * A.stage_bytes;
        constexpr uint32_t E = sizeof(T);
        const uint32_t ia_b = st_s + lay.o_ia + 4u * offs[s][0];
        const uint32_t ad_b = st_s + lay.o_ad + E * offs[s][1];
        const uint32_t ja_b0 = st_s + lay.o_ja + 4u * offs[s][2];
        const uint32_t al_b0 = st_s + lay.o_al + E * offs[s][3];
        const uint32_t au_b0 = sym ? al_b0 : st_s + lay.o_au + E * offs[s][4];
        const int32_t p0 = lds_i(ia_b);

        const bool act = row < nr;
        const int32_t g = g0 + row;
        T yi = T(0), xi = T(0);
        if (act) {
            xi = __ldg(xb + g);
            const int32_t rb = lds_i(ia_b + 4u * row) - p0;
            const int32_t len = lds_i(ia_b + 4u * (row + 1)) - p0 - rb;
            // L = 1: the lane's slots in a batch are strided by nb, so the slot
            // pairs neighbouring rows share (d, d+1) never meet in a batch.
            // L > 1: sub-lane sub owns the blocked slot range [sub*q, sub*q+m)
            // (one instruction never pairs d with d+1 across neighbouring rows)
            const int32_t q = L == 1 ? len : (len + L - 1) / L;
            const int32_t first = rb + sub * q;
            const int32_t m = L == 1 ? len : max(0, min(q, len - sub * q));
            const int32_t nb = (m + 3) >> 2;
            const uint32_t ja_b = ja_b0 + 4u * first;
            const uint32_t al_b = al_b0 + E * first;
            const uint32_t au_b = au_b0 + E * first;
            // rotated batch order (A.rotate): consecutive rows start on different
            // batches, so rows sharing their column lists (3x3 dof blocks) do not
            // hit the same scatter targets at the same time
            const int32_t rot = A.rotate > 1 && nb > 1 ? (g % A.rotate) % nb : 0;
            // scatter combining (A.combine, ring-free only): every row's slots rotated by
            // -g (mod m), so in one instruction neighbouring rows r, r+1 visit slots s and
            // s-1 -- the same target whenever their offsets differ by one (stencil
            // families) -- and lanes with equal targets add into one red.global
            const bool comb = !RINGS && A.combine;
            const int32_t gm = comb && m > 0 ? g % m : 0;
            for (int32_t bi = 0; bi < nb; ++bi) {
                const int32_t bt = bi + rot < nb ? bi + rot : bi + rot - nb;
                int32_t mm[4], j[4];
                T xv[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    mm[u] = L == 1 ? bt + u * nb : 4 * bt + u;
                    if (comb && mm[u] < m) mm[u] = mm[u] >= gm ? mm[u] - gm : mm[u] + m - gm;
                    j[u] = mm[u] < m ? lds_i(ja_b + 4u * mm[u]) : -1;
                }
#pragma unroll
                for (int u = 0; u < 4; ++u) xv[u] = j[u] >= 0 ? __ldg(xb + j[u]) : T(0);
                uint32_t sa[4];
                T val[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    sa[u] = 0u;
                    val[u] = T(0);
                    if (j[u] >= 0) {
                        yi = fma(lds_f(al_b + E * mm[u], T(0)), xv[u], yi);
                        val[u] = lds_f(au_b + E * mm[u], T(0)) * xi;
                        if (!RINGS) {
                            if (!comb) red_add((j[u] < rs ? sp : out) + j[u], val[u]);
                            continue;
                        }
                        const int32_t d = g - j[u];
                        if (d <= near_depth)
                            sa[u] = ringN_s + E * static_cast<uint32_t>(j[u] & maskN);
                        else if (static_cast<uint32_t>(d - far_lo) <= far_span && far_on)
                            sa[u] = ringF_s + E * static_cast<uint32_t>(j[u] & maskF);
                        else
                            red_add(out + j[u], val[u]);
                    }
                }
                if (!RINGS) {
                    if (comb) {
                        const unsigned am = __activemask();
#pragma unroll
                        for (int u = 0; u < 4; ++u) {
                            const unsigned grp = __match_any_sync(am, j[u]);
                            const int cnt = __popc(grp);
                            const int mx = __reduce_max_sync(am, cnt);
                            T tot = T(0);
                            unsigned rest = grp;
                            for (int k = 0; k < mx; ++k) {  // the k-th member's value, lane order
                                const int src = rest ? __ffs(rest) - 1 : lane;
                                const T o = __shfl_sync(am, val[u], src);
                                if (rest) tot += o;
                                rest &= rest - 1u;
                            }
                            if (j[u] >= 0 && lane == __ffs(grp) - 1)
                                red_add((j[u] < rs ? sp : out) + j[u], tot);
                        }
                    }
                    continue;
                }
                if (L == 1) {
                    T old[4];  // four independent CAS in flight
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
                } else {
                    // consecutive slots of one lane may pair d with d+1 across
                    // rows: read each old value right before its CAS
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        if (!sa[u]) continue;
                        T o = lds_f(sa[u], T(0));
                        T seen = cas_s(sa[u], o, o + val[u]);
                        while (!same_bits(seen, o)) {
                            o = seen;
                            seen = cas_s(sa[u], o, o + val[u]);
                        }
                    }
                }
            }
        }
        // all lanes reach the width-L reduction (rows >= nr contribute 0)
#pragma unroll
        for (int off = L / 2; off > 0; off >>= 1) yi += __shfl_xor_sync(0xffffffffu, yi, off, L);
        if (!RINGS && act && sub == 0) red_add(out + g, yi + lds_f(ad_b + E * row, T(0)) * xi);
        if (RINGS && act && sub == 0) {
            const uint32_t a = ringN_s + static_cast<uint32_t>(g & maskN) * sizeof(T);
            const T add = yi + lds_f(ad_b + E * row, T(0)) * xi;
            T old0 = lds_f(a, T(0));
            T seen = cas_s(a, old0, old0 + add);
            while (!same_bits(seen, old0)) {
                old0 = seen;
                seen = cas_s(a, old0, old0 + add);
            }
        }
        // mbarrier arrive has release semantics for this warp's shared-memory
        // updates (ordered by __syncwarp); no MEMBAR that would also wait for
        // the flush's outstanding red.global ops
        __syncwarp();
        if (lane == 0) {
            mbar_arrive(&empty[s]);                   // stage s may be refilled
            if (RINGS) mbar_arrive(&done[ti % kDoneSlots]);  // tile ti's ring contributions are in
        }
    }
    // the last tile's flush
    const int tl = t_count - 1;
    if (RINGS && tl % kConsumerWarps == cw) {
        mbar_wait(&done[tl % kDoneSlots], (tl / kDoneSlots) & 1);
        flush_tile(A, out, rings, bank_elems, dring[tl % kDoneSlots], lane);
    }
}

}  // namespace dev
}  // namespace csrcgpu

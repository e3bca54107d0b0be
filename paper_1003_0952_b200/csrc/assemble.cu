// Device CSRC construction: build_csr (csr.hpp:55-92), csr_to_csrc
// (csrc_matrix.hpp:44-91), decompose_rect (csrc_matrix.hpp:113-142) on the GPU.
//
// The reference builds CSRC on one host core by sorting an index array of the
// triplets with std::sort on (row, col), summing duplicates in sorted order,
// then looking every lower entry's transpose up with a binary search
// (csrc_matrix.hpp:61-66). Here the same three steps are device passes over
// HBM-resident arrays:
//
//   1. bounds check          one pass, atomicMin of the first offending entry
//                            (the reference throws on the first in input order)
//   2. sort + reduce         key = row << cb | col (cb = bits of n_cols),
//                            stable LSD radix sort of (key, entry id); a head
//                            flag + exclusive scan numbers the unique (row, col)
//                            pairs; each run's head sums its duplicates in
//                            stable (input) order, as build_csr's
//                            `values.back() += e.value` does in sorted order;
//                            row_ptr by a lower_bound per row over the keys.
//   3. csr -> csrc           per row: lower count + diagonal (lower_bound of i
//                            in the sorted row); ia by an exclusive scan; per
//                            entry: transpose lookup by binary search in row j,
//                            ja/al/au written in CSR order (= CSRC order), the
//                            exact value-symmetry test (upper != lower), and the
//                            first error in the reference's row-major order.
//
// Bit-exactness: every output value is a copy of an input value or a sum of
// duplicates in input order; the reference sums them in its std::sort order,
// which equals input order for pairs (a + b == b + a) and for every run of
// equal keys that introsort leaves in input order. Tests compare against the
// compiled reference (tests/test_gpu_assemble.py).
//
// Sizes: C5 (449 M triplets) needs ~31 GB of HBM (triplets 7.2 GB, keys and
// ids double-buffered 10.8 GB, CSR 7.2 GB, CSRC 4.8 GB).
#include <cuda_runtime.h>

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <chrono>
#include <memory>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "hostlink.cuh"
#include "internal.hpp"

using namespace csrcgpu;


struct csrc_built_s {
    // CSR (build_csr) and/or CSRC (csr_to_csrc); host arrays owned here
    int has_csr = 0, has_csrc = 0;
    index_t n_rows = 0, n_cols = 0;
    HVec<index_t> row_ptr, col_idx;
    HVec<double> values;
    index_t n = 0;
    HVec<double> ad, al, au;
    HVec<index_t> ia, ja;
    int value_symmetric = 0;
    // rectangular tail (decompose_rect): CSR over columns n..m-1, local indices
    int has_rect = 0;
    index_t m_cols = 0;
    HVec<index_t> t_row_ptr, t_col_idx;
    HVec<double> t_values;
    double ms[4] = {0, 0, 0, 0};  // h2d, sort+reduce, convert, d2h
};

namespace {

#define ACUDA(expr)                                                                     \
    do {                                                                                \
        cudaError_t _e = (expr);                                                        \
        if (_e != cudaSuccess)                                                          \
            throw Error(std::string("CUDA error: ") + cudaGetErrorString(_e) + " at " + \
                        #expr);                                                         \
    } while (0)

constexpr unsigned long long kNone = ~0ull;

// Scoped device allocation (freed on every exit path, so errors thrown
// mid-build do not leak HBM).
struct DMem {
    void* p = nullptr;
    DMem() = default;
    explicit DMem(size_t bytes) { alloc(bytes); }
    DMem(const DMem&) = delete;
    DMem& operator=(const DMem&) = delete;
    ~DMem() { release(); }
    void alloc(size_t bytes) {
        release();
        ACUDA(cudaMalloc(&p, std::max<size_t>(bytes, 16)));
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
    }
    template <class U>
    U* as() const { return static_cast<U*>(p); }
};

struct Clock {
    std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
    double lap() {
        auto t = std::chrono::steady_clock::now();
        double ms = std::chrono::duration<double, std::milli>(t - t0).count();
        t0 = t;
        return ms;
    }
};

int bits_for(int64_t v) {  // bits needed to hold 0..v-1
    int b = 0;
    while ((int64_t{1} << b) < v) ++b;
    return std::max(b, 1);
}

unsigned grid_for(int64_t items, int threads = 256) {
    int64_t g = (items + threads - 1) / threads;
    return static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>(g, 1 << 30)));
}

// ---------------------------------------------------------------- kernels
__global__ void k_bounds(int64_t m, const index_t* __restrict__ r, const index_t* __restrict__ c,
                         index_t n_rows, index_t n_cols, unsigned long long* first_bad) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m;
         e += (int64_t)gridDim.x * blockDim.x) {
        const index_t row = r[e], col = c[e];
        if (row < 0 || row >= n_rows || col < 0 || col >= n_cols)
            atomicMin(first_bad, static_cast<unsigned long long>(e));
    }
}

__global__ void k_keys(int64_t m, const index_t* __restrict__ r, const index_t* __restrict__ c,
                       int cb, unsigned long long* __restrict__ key, uint32_t* __restrict__ id) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m;
         e += (int64_t)gridDim.x * blockDim.x) {
        key[e] = (static_cast<unsigned long long>(r[e]) << cb) | static_cast<uint32_t>(c[e]);
        id[e] = static_cast<uint32_t>(e);
    }
}

__global__ void k_heads(int64_t m, const unsigned long long* __restrict__ key,
                        uint32_t* __restrict__ head) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m;
         e += (int64_t)gridDim.x * blockDim.x)
        head[e] = (e == 0 || key[e] != key[e - 1]) ? 1u : 0u;
}

// One thread per run head: the CSR entry = the run's (row, col), its value the
// duplicates summed left to right in stable (input) order (csr.hpp:77-88).
__global__ void k_emit(int64_t m, const unsigned long long* __restrict__ key,
                       const uint32_t* __restrict__ id, const uint32_t* __restrict__ head,
                       const uint32_t* __restrict__ pos, const double* __restrict__ v, int cb,
                       index_t* __restrict__ col, double* __restrict__ val,
                       index_t* __restrict__ erow) {
    const unsigned long long cmask = (1ull << cb) - 1;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m;
         e += (int64_t)gridDim.x * blockDim.x) {
        if (!head[e]) continue;
        const unsigned long long k = key[e];
        double s = v[id[e]];
        for (int64_t f = e + 1; f < m && key[f] == k; ++f) s += v[id[f]];
        const uint32_t q = pos[e];
        col[q] = static_cast<index_t>(k & cmask);
        val[q] = s;
        erow[q] = static_cast<index_t>(k >> cb);
    }
}

// row_ptr[i] = number of unique entries of rows < i (lower_bound of i << cb).
__global__ void k_rowptr(int64_t m, const unsigned long long* __restrict__ key,
                         const uint32_t* __restrict__ pos, uint32_t nnz, index_t n_rows, int cb,
                         index_t* __restrict__ row_ptr) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i <= n_rows;
         i += (int64_t)gridDim.x * blockDim.x) {
        const unsigned long long target = static_cast<unsigned long long>(i) << cb;
        int64_t lo = 0, hi = m;
        while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if (key[mid] < target) lo = mid + 1; else hi = mid;
        }
        row_ptr[i] = lo < m ? static_cast<index_t>(pos[lo]) : static_cast<index_t>(nnz);
    }
}

// erow for a caller-supplied CSR (csr_to_csrc entry point).
__global__ void k_erow(index_t n, const index_t* __restrict__ rp, index_t* __restrict__ erow) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        for (index_t k = rp[i]; k < rp[i + 1]; ++k) erow[k] = static_cast<index_t>(i);
}

__device__ __forceinline__ index_t lower_bound_dev(const index_t* __restrict__ a, index_t lo,
                                                   index_t hi, index_t x) {
    while (lo < hi) {
        const index_t mid = lo + ((hi - lo) >> 1);
        if (a[mid] < x) lo = mid + 1; else hi = mid;
    }
    return lo;
}

// Per row: lower count (entries with col < i) and the diagonal. A missing
// diagonal is reported after the row's entries (csrc_matrix.hpp:79-81): error
// order key 2*row_ptr[i+1]-1, between the row's last entry (2k) and the next
// row's first.
__global__ void k_rows(index_t n, const index_t* __restrict__ rp, const index_t* __restrict__ col,
                       const double* __restrict__ val, index_t* __restrict__ lcnt,
                       double* __restrict__ ad, unsigned long long* first_err) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const index_t b = rp[i], e = rp[i + 1];
        const index_t d = lower_bound_dev(col, b, e, static_cast<index_t>(i));
        lcnt[i] = d - b;
        if (d < e && col[d] == i) {
            ad[i] = val[d];
        } else {
            ad[i] = 0.0;
            const unsigned long long okey = 2ull * static_cast<unsigned long long>(e) - 1ull;
            atomicMin(first_err, (okey << 32) | static_cast<unsigned long long>(i));
        }
    }
}

// Per CSR entry (i, j): lower entries go to CSRC position ia[i] + (k - rp[i])
// with the transpose looked up in row j; upper entries only check theirs.
__global__ void k_csrc(int64_t nnz, const index_t* __restrict__ rp, const index_t* __restrict__ col,
                       const double* __restrict__ val, const index_t* __restrict__ erow,
                       const index_t* __restrict__ ia, index_t* __restrict__ ja,
                       double* __restrict__ al, double* __restrict__ au,
                       unsigned long long* first_err, int* asym) {
    int local_asym = 0;
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < nnz;
         k += (int64_t)gridDim.x * blockDim.x) {
        const index_t i = erow[k], j = col[k];
        if (j == i) continue;
        const index_t jb = rp[j], je = rp[j + 1];
        const index_t t = lower_bound_dev(col, jb, je, i);
        const bool found = t < je && col[t] == i;
        if (!found) {
            const unsigned long long okey = 2ull * static_cast<unsigned long long>(k);
            atomicMin(first_err, (okey << 32) | static_cast<unsigned long long>(i));
            continue;
        }
        if (j < i) {
            const index_t q = ia[i] + static_cast<index_t>(k - rp[i]);
            const double lv = val[k], uv = val[t];
            ja[q] = j;
            al[q] = lv;
            au[q] = uv;
            if (uv != lv) local_asym = 1;  // exact test, NaN counts as a mismatch (:70)
        }
    }
    if (local_asym) atomicOr(asym, 1);
}

// ------------------------------------------------------------- helpers
template <class T>
void h2d(HostLink& hl, DMem& d, const T* h, int64_t count) {
    d.alloc(static_cast<size_t>(count) * sizeof(T));
    if (count) hl.h2d(d.p, h, static_cast<size_t>(count) * sizeof(T));
}

template <class T>
void d2h(HostLink& hl, HVec<T>& h, const DMem& d, int64_t count) {
    h.resize(static_cast<size_t>(count));
    if (count) hl.d2h(h.data(), d.p, static_cast<size_t>(count) * sizeof(T));
}

unsigned long long read_u64(const DMem& d) {
    unsigned long long v = 0;
    ACUDA(cudaMemcpy(&v, d.p, sizeof(v), cudaMemcpyDeviceToHost));
    return v;
}

// Device CSR, the output of the sort + reduce stage.
struct DevCsr {
    index_t n_rows = 0, n_cols = 0;
    int64_t nnz = 0;
    DMem rp, col, val, erow;
};

// build_csr (csr.hpp:55-92) on device-resident triplets.
void build_csr_dev(index_t n_rows, index_t n_cols, int64_t m, const DMem& r, const DMem& c,
                   const DMem& v, DevCsr& out, bool want_erow, cudaStream_t st, double* ms_sort) {
    Clock clk;
    out.n_rows = n_rows;
    out.n_cols = n_cols;
    out.rp.alloc((static_cast<size_t>(n_rows) + 1) * sizeof(index_t));
    if (m == 0) {
        ACUDA(cudaMemsetAsync(out.rp.p, 0, (static_cast<size_t>(n_rows) + 1) * sizeof(index_t), st));
        out.nnz = 0;
        out.col.alloc(16);
        out.val.alloc(16);
        out.erow.alloc(16);
        ACUDA(cudaStreamSynchronize(st));
        *ms_sort += clk.lap();
        return;
    }
    const int cb = bits_for(n_cols);
    const int rb = bits_for(static_cast<int64_t>(n_rows));
    DMem key0(m * 8), key1(m * 8), id0(m * 4), id1(m * 4);
    k_keys<<<grid_for(m), 256, 0, st>>>(m, r.as<index_t>(), c.as<index_t>(), cb,
                                         key0.as<unsigned long long>(), id0.as<uint32_t>());
    ACUDA(cudaGetLastError());
    cub::DoubleBuffer<unsigned long long> kb(key0.as<unsigned long long>(), key1.as<unsigned long long>());
    cub::DoubleBuffer<uint32_t> vb(id0.as<uint32_t>(), id1.as<uint32_t>());
    size_t tmp_bytes = 0;
    ACUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, kb, vb, static_cast<int>(m), 0, cb + rb, st));
    {
        DMem tmp(tmp_bytes);
        ACUDA(cub::DeviceRadixSort::SortPairs(tmp.p, tmp_bytes, kb, vb, static_cast<int>(m), 0, cb + rb, st));
        ACUDA(cudaStreamSynchronize(st));
    }
    const unsigned long long* key = kb.Current();
    const uint32_t* id = vb.Current();
    // head flags into the spare key buffer's storage, positions into the spare id buffer
    uint32_t* head = reinterpret_cast<uint32_t*>(kb.Alternate());
    uint32_t* pos = vb.Alternate();
    k_heads<<<grid_for(m), 256, 0, st>>>(m, key, head);
    ACUDA(cudaGetLastError());
    tmp_bytes = 0;
    ACUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, head, pos, static_cast<int>(m), st));
    {
        DMem tmp(tmp_bytes);
        ACUDA(cub::DeviceScan::ExclusiveSum(tmp.p, tmp_bytes, head, pos, static_cast<int>(m), st));
        ACUDA(cudaStreamSynchronize(st));
    }
    uint32_t last_pos = 0, last_head = 0;
    ACUDA(cudaMemcpy(&last_pos, pos + (m - 1), 4, cudaMemcpyDeviceToHost));
    ACUDA(cudaMemcpy(&last_head, head + (m - 1), 4, cudaMemcpyDeviceToHost));
    const uint32_t nnz = last_pos + last_head;
    out.nnz = nnz;
    out.col.alloc(static_cast<size_t>(nnz) * 4);
    out.val.alloc(static_cast<size_t>(nnz) * 8);
    out.erow.alloc(static_cast<size_t>(nnz) * 4);
    k_emit<<<grid_for(m), 256, 0, st>>>(m, key, id, head, pos, v.as<double>(), cb, out.col.as<index_t>(),
                                         out.val.as<double>(), out.erow.as<index_t>());
    ACUDA(cudaGetLastError());
    k_rowptr<<<grid_for(static_cast<int64_t>(n_rows) + 1), 256, 0, st>>>(m, key, pos, nnz, n_rows, cb,
                                                                          out.rp.as<index_t>());
    ACUDA(cudaGetLastError());
    ACUDA(cudaStreamSynchronize(st));
    if (!want_erow) out.erow.release();
    *ms_sort += clk.lap();
}

void check_bounds(index_t n_rows, index_t n_cols, int64_t m, const DMem& r, const DMem& c,
                  const index_t* rows_h, const index_t* cols_h, cudaStream_t st) {
    if (m == 0) return;
    DMem bad(8);
    ACUDA(cudaMemsetAsync(bad.p, 0xff, 8, st));
    k_bounds<<<grid_for(m), 256, 0, st>>>(m, r.as<index_t>(), c.as<index_t>(), n_rows, n_cols,
                                           bad.as<unsigned long long>());
    ACUDA(cudaGetLastError());
    ACUDA(cudaStreamSynchronize(st));
    const unsigned long long e = read_u64(bad);
    if (e != kNone)
        throw Error("build_csr: entry (" + std::to_string(rows_h[e]) + ", " + std::to_string(cols_h[e]) +
                    ") outside " + std::to_string(n_rows) + "x" + std::to_string(n_cols) + " bounds");
}

// csr_to_csrc (csrc_matrix.hpp:44-91) on a device CSR with erow.
void csr_to_csrc_dev(const DevCsr& a, csrc_built_s& out, cudaStream_t st, HostLink& hl, double* ms_conv,
                     double* ms_d2h) {
    Clock clk;
    if (a.n_rows != a.n_cols) throw Error("csr_to_csrc: matrix is not square");
    const index_t n = a.n_rows;
    DMem lcnt((static_cast<size_t>(n) + 1) * 4), ia((static_cast<size_t>(n) + 1) * 4), ad(static_cast<size_t>(n) * 8);
    DMem err(8), asym(4);
    ACUDA(cudaMemsetAsync(err.p, 0xff, 8, st));
    ACUDA(cudaMemsetAsync(asym.p, 0, 4, st));
    ACUDA(cudaMemsetAsync(lcnt.as<index_t>() + n, 0, 4, st));
    if (n > 0) {
        k_rows<<<grid_for(n), 256, 0, st>>>(n, a.rp.as<index_t>(), a.col.as<index_t>(), a.val.as<double>(),
                                             lcnt.as<index_t>(), ad.as<double>(), err.as<unsigned long long>());
        ACUDA(cudaGetLastError());
    }
    size_t tmp_bytes = 0;
    ACUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, lcnt.as<index_t>(), ia.as<index_t>(), n + 1, st));
    {
        DMem tmp(tmp_bytes);
        ACUDA(cub::DeviceScan::ExclusiveSum(tmp.p, tmp_bytes, lcnt.as<index_t>(), ia.as<index_t>(), n + 1, st));
        ACUDA(cudaStreamSynchronize(st));
    }
    index_t k = 0;
    ACUDA(cudaMemcpy(&k, ia.as<index_t>() + n, 4, cudaMemcpyDeviceToHost));
    DMem ja(static_cast<size_t>(k) * 4), al(static_cast<size_t>(k) * 8), au(static_cast<size_t>(k) * 8);
    if (a.nnz > 0) {
        k_csrc<<<grid_for(a.nnz), 256, 0, st>>>(a.nnz, a.rp.as<index_t>(), a.col.as<index_t>(), a.val.as<double>(),
                                                 a.erow.as<index_t>(), ia.as<index_t>(), ja.as<index_t>(),
                                                 al.as<double>(), au.as<double>(), err.as<unsigned long long>(),
                                                 asym.as<int>());
        ACUDA(cudaGetLastError());
    }
    ACUDA(cudaStreamSynchronize(st));
    *ms_conv += clk.lap();
    const unsigned long long code = read_u64(err);
    if (code != kNone) {
        const unsigned long long okey = code >> 32;
        const index_t row = static_cast<index_t>(code & 0xffffffffull);
        if (okey & 1ull) throw Error("csr_to_csrc: row " + std::to_string(row) + " has no diagonal entry");
        const int64_t kk = static_cast<int64_t>(okey >> 1);
        index_t j = 0;
        ACUDA(cudaMemcpy(&j, a.col.as<index_t>() + kk, 4, cudaMemcpyDeviceToHost));
        throw Error("csr_to_csrc: entry (" + std::to_string(row) + ", " + std::to_string(j) +
                    ") has no transpose (" + std::to_string(j) + ", " + std::to_string(row) + ")");
    }
    int asym_h = 0;
    ACUDA(cudaMemcpy(&asym_h, asym.p, 4, cudaMemcpyDeviceToHost));
    out.has_csrc = 1;
    out.n = n;
    out.value_symmetric = asym_h ? 0 : 1;
    d2h(hl, out.ad, ad, n);
    d2h(hl, out.ia, ia, static_cast<int64_t>(n) + 1);
    d2h(hl, out.ja, ja, k);
    d2h(hl, out.al, al, k);
    if (!out.value_symmetric) d2h(hl, out.au, au, k);
    else out.au.clear();
    *ms_d2h += clk.lap();
}

void csr_to_host(HostLink& hl, const DevCsr& a, HVec<index_t>& rp, HVec<index_t>& col, HVec<double>& val) {
    d2h(hl, rp, a.rp, static_cast<int64_t>(a.n_rows) + 1);
    d2h(hl, col, a.col, a.nnz);
    d2h(hl, val, a.val, a.nnz);
}

struct DeviceScope {
    int prev = 0;
    explicit DeviceScope(int dev) {
        int count = 0;
        if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0)
            throw Error("no CUDA device available (the product has no CPU path)");
        if (dev < 0 || dev >= count) throw Error("device " + std::to_string(dev) + " out of range");
        cudaGetDevice(&prev);
        ACUDA(cudaSetDevice(dev));
    }
    ~DeviceScope() { cudaSetDevice(prev); }
};

struct Stream {
    cudaStream_t s = nullptr;
    Stream() { ACUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking)); }
    ~Stream() { cudaStreamDestroy(s); }
};

void check_triplets(int64_t m, const int32_t* rows, const int32_t* cols, const double* vals) {
    if (m < 0) throw Error("build_csr: negative triplet count");
    if (m > 0 && (!rows || !cols || !vals)) throw Error("build_csr: null triplet array");
    if (m >= (int64_t{1} << 31) - 1)
        throw Error("build_csr: " + std::to_string(m) + " triplets exceed the 2^31-1 entries of csrc::index_t");
}

}  // namespace

extern "C" {

int csrc_gpu_build_csr(int32_t n_rows, int32_t n_cols, int64_t m, const int32_t* rows,
                       const int32_t* cols, const double* vals, int32_t device, csrc_built_t* out) {
    return guarded(__func__, [&] {
        if (!out) throw Error("build_csr: null output handle");
        *out = nullptr;
        if (n_rows < 0 || n_cols < 0) throw Error("build_csr: negative dimensions");
        check_triplets(m, rows, cols, vals);
        DeviceScope ds(device);
        Stream st;
        auto b = std::make_unique<csrc_built_s>();
        HostLink hl(st.s);
        Clock clk;
        DMem r, c, v;
        h2d(hl, r, rows, m);
        h2d(hl, c, cols, m);
        h2d(hl, v, vals, m);
        b->ms[0] = clk.lap();
        check_bounds(n_rows, n_cols, m, r, c, rows, cols, st.s);
        DevCsr csr;
        build_csr_dev(n_rows, n_cols, m, r, c, v, csr, false, st.s, &b->ms[1]);
        clk.lap();
        b->has_csr = 1;
        b->n_rows = n_rows;
        b->n_cols = n_cols;
        csr_to_host(hl, csr, b->row_ptr, b->col_idx, b->values);
        b->ms[3] = clk.lap();
        *out = b.release();
    });
}

int csrc_gpu_build_csrc(int32_t n, int64_t m, const int32_t* rows, const int32_t* cols,
                        const double* vals, int32_t device, csrc_built_t* out) {
    return guarded(__func__, [&] {
        if (!out) throw Error("build_csr: null output handle");
        *out = nullptr;
        if (n < 0) throw Error("build_csr: negative dimensions");
        check_triplets(m, rows, cols, vals);
        DeviceScope ds(device);
        Stream st;
        auto b = std::make_unique<csrc_built_s>();
        HostLink hl(st.s);
        Clock clk;
        DMem r, c, v;
        h2d(hl, r, rows, m);
        h2d(hl, c, cols, m);
        h2d(hl, v, vals, m);
        b->ms[0] = clk.lap();
        check_bounds(n, n, m, r, c, rows, cols, st.s);
        DevCsr csr;
        build_csr_dev(n, n, m, r, c, v, csr, true, st.s, &b->ms[1]);
        r.release();
        c.release();
        v.release();
        csr_to_csrc_dev(csr, *b, st.s, hl, &b->ms[2], &b->ms[3]);
        *out = b.release();
    });
}

int csrc_gpu_csr_to_csrc(int32_t n_rows, int32_t n_cols, const int32_t* row_ptr,
                         const int32_t* col_idx, const double* values, int32_t device,
                         csrc_built_t* out) {
    return guarded(__func__, [&] {
        if (!out) throw Error("csr_to_csrc: null output handle");
        *out = nullptr;
        if (n_rows != n_cols) throw Error("csr_to_csrc: matrix is not square");
        if (n_rows < 0 || !row_ptr) throw Error("csr_to_csrc: invalid row pointers");
        const int64_t nnz = row_ptr[n_rows];
        if (nnz > 0 && (!col_idx || !values)) throw Error("csr_to_csrc: null column or value array");
        DeviceScope ds(device);
        Stream st;
        auto b = std::make_unique<csrc_built_s>();
        HostLink hl(st.s);
        Clock clk;
        DevCsr csr;
        csr.n_rows = n_rows;
        csr.n_cols = n_cols;
        csr.nnz = nnz;
        h2d(hl, csr.rp, row_ptr, static_cast<int64_t>(n_rows) + 1);
        h2d(hl, csr.col, col_idx, nnz);
        h2d(hl, csr.val, values, nnz);
        csr.erow.alloc(static_cast<size_t>(nnz) * 4);
        b->ms[0] = clk.lap();
        if (n_rows > 0) {
            k_erow<<<grid_for(n_rows), 256, 0, st.s>>>(n_rows, csr.rp.as<index_t>(), csr.erow.as<index_t>());
            ACUDA(cudaGetLastError());
        }
        csr_to_csrc_dev(csr, *b, st.s, hl, &b->ms[2], &b->ms[3]);
        *out = b.release();
    });
}

int csrc_gpu_decompose_rect(int32_t n_rows, int32_t n_cols, const int32_t* row_ptr,
                            const int32_t* col_idx, const double* values, int32_t device,
                            csrc_built_t* out) {
    return guarded(__func__, [&] {
        if (!out) throw Error("decompose_rect: null output handle");
        *out = nullptr;
        if (n_cols <= n_rows)
            throw Error("decompose_rect: requires n_cols > n_rows (got " + std::to_string(n_rows) + "x" +
                        std::to_string(n_cols) + ")");
        if (!row_ptr) throw Error("decompose_rect: invalid row pointers");
        const index_t n = n_rows;
        // split on the host (one pass over the CSR), as csrc_matrix.hpp:123-132
        std::vector<index_t> lr, lc, tr, tc;
        std::vector<double> lv, tv;
        for (index_t i = 0; i < n; ++i)
            for (index_t k = row_ptr[i]; k < row_ptr[i + 1]; ++k) {
                const index_t j = col_idx[k];
                if (j < n) {
                    lr.push_back(i);
                    lc.push_back(j);
                    lv.push_back(values[k]);
                } else {
                    tr.push_back(i);
                    tc.push_back(j - n);
                    tv.push_back(values[k]);
                }
            }
        csrc_built_t lead = nullptr, tail = nullptr;
        if (csrc_gpu_build_csrc(n, static_cast<int64_t>(lr.size()), lr.data(), lc.data(), lv.data(), device, &lead))
            throw Error(csrc_gpu_last_error());
        std::unique_ptr<csrc_built_s> b(lead);
        if (csrc_gpu_build_csr(n, n_cols - n, static_cast<int64_t>(tr.size()), tr.data(), tc.data(), tv.data(),
                               device, &tail))
            throw Error(csrc_gpu_last_error());
        std::unique_ptr<csrc_built_s> t(tail);
        b->has_rect = 1;
        b->m_cols = n_cols;
        b->t_row_ptr = std::move(t->row_ptr);
        b->t_col_idx = std::move(t->col_idx);
        b->t_values = std::move(t->values);
        for (int q = 0; q < 4; ++q) b->ms[q] += t->ms[q];
        *out = b.release();
    });
}

int csrc_built_matrix(csrc_built_t b, csrc_host_matrix* m) {
    return guarded(__func__, [&] {
        if (!b || !m) throw Error("csrc_built_matrix: null argument");
        if (!b->has_csrc) throw Error("csrc_built_matrix: handle holds no CSRC matrix");
        m->n = b->n;
        m->k = static_cast<int64_t>(b->ja.size());
        m->ad = b->ad.data();
        m->ia = b->ia.data();
        m->ja = b->ja.data();
        m->al = b->al.data();
        m->au = b->value_symmetric ? nullptr : b->au.data();
        m->value_symmetric = b->value_symmetric;
    });
}

int csrc_built_csr(csrc_built_t b, int32_t* n_rows, int32_t* n_cols, int64_t* nnz,
                   const int32_t** row_ptr, const int32_t** col_idx, const double** values) {
    return guarded(__func__, [&] {
        if (!b) throw Error("csrc_built_csr: null handle");
        if (!b->has_csr) throw Error("csrc_built_csr: handle holds no CSR matrix");
        *n_rows = b->n_rows;
        *n_cols = b->n_cols;
        *nnz = static_cast<int64_t>(b->values.size());
        *row_ptr = b->row_ptr.data();
        *col_idx = b->col_idx.data();
        *values = b->values.data();
    });
}

int csrc_built_rect_tail(csrc_built_t b, int32_t* m_cols, int64_t* nnz, const int32_t** row_ptr,
                         const int32_t** col_idx, const double** values) {
    return guarded(__func__, [&] {
        if (!b) throw Error("csrc_built_rect_tail: null handle");
        if (!b->has_rect) throw Error("csrc_built_rect_tail: handle holds no rectangular tail");
        *m_cols = b->m_cols;
        *nnz = static_cast<int64_t>(b->t_values.size());
        *row_ptr = b->t_row_ptr.data();
        *col_idx = b->t_col_idx.data();
        *values = b->t_values.data();
    });
}

int csrc_built_timings(csrc_built_t b, double* ms4) {
    return guarded(__func__, [&] {
        if (!b || !ms4) throw Error("csrc_built_timings: null argument");
        for (int q = 0; q < 4; ++q) ms4[q] = b->ms[q];
    });
}

void csrc_built_free(csrc_built_t b) { delete b; }

}  // extern "C"

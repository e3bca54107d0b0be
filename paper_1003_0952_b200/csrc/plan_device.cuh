// Device-side transposition of CSRC pairs into per-row gather entry streams
// (capi.cu setup_gather, whole-matrix plans): the same layout the host
// builder produces -- row q's lower pairs in CSRC order, then the pairs that
// name q as their column in ascending source row -- built with a stable radix
// sort of the pairs by column instead of a host pass over 400 M pairs.
#pragma once

#include <cstdint>

namespace csrcgpu {
namespace dev {

__global__ void k_iota(int64_t k, int32_t* __restrict__ v) {
    for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < k;
         t += static_cast<int64_t>(gridDim.x) * blockDim.x)
        v[t] = static_cast<int32_t>(t);
}

// erow[t] = the row of pair t
__global__ void k_pair_rows(int32_t n, const int32_t* __restrict__ ia, int32_t* __restrict__ erow) {
    for (int64_t q = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; q < n;
         q += static_cast<int64_t>(gridDim.x) * blockDim.x)
        for (int32_t t = ia[q]; t < ia[q + 1]; ++t) erow[t] = static_cast<int32_t>(q);
}

// cnt[q] = lower pairs of q + pairs naming q (upper counts by atomics)
__global__ void k_upper_counts(int64_t k, const int32_t* __restrict__ ja, int32_t* __restrict__ up) {
    for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < k;
         t += static_cast<int64_t>(gridDim.x) * blockDim.x)
        atomicAdd(up + ja[t], 1);
}

__global__ void k_row_counts(int32_t n, const int32_t* __restrict__ ia, const int32_t* __restrict__ up,
                             int32_t* __restrict__ cnt) {
    for (int64_t q = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; q < n;
         q += static_cast<int64_t>(gridDim.x) * blockDim.x)
        cnt[q] = (ia[q + 1] - ia[q]) + up[q];
}

// lower pairs at eptr[q] + (t - ia[q])
__global__ void k_place_lower(int64_t k, const int32_t* __restrict__ erow, const int32_t* __restrict__ ia,
                              const int32_t* __restrict__ ja, const double* __restrict__ al,
                              const double* __restrict__ au, const int32_t* __restrict__ eptr,
                              int32_t* __restrict__ eidx, double* __restrict__ ev, double* __restrict__ evt) {
    for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < k;
         t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int32_t q = erow[t];
        const int64_t pos = eptr[q] + (t - ia[q]);
        eidx[pos] = ja[t];
        ev[pos] = al[t];
        if (evt) evt[pos] = au[t];
    }
}

// upper pairs: sorted index i (pairs stably sorted by column) -> column q =
// key[i], pair t = val[i]; its rank among the pairs naming q is i - ustart[q]
__global__ void k_place_upper(int64_t k, const int32_t* __restrict__ key, const int32_t* __restrict__ val,
                              const int32_t* __restrict__ ustart, const int32_t* __restrict__ ia,
                              const int32_t* __restrict__ erow, const double* __restrict__ al,
                              const double* __restrict__ au, const int32_t* __restrict__ eptr,
                              int32_t* __restrict__ eidx, double* __restrict__ ev, double* __restrict__ evt) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < k;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int32_t q = key[i], t = val[i];
        const int64_t pos = eptr[q] + (ia[q + 1] - ia[q]) + (i - ustart[q]);
        eidx[pos] = erow[t];
        ev[pos] = au ? au[t] : al[t];
        if (evt) evt[pos] = al[t];
    }
}

}  // namespace dev
}  // namespace csrcgpu

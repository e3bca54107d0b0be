// Multi-GPU band executor behind the C ABI: one per rank (one process per GPU),
// owning an NCCL communicator. Rank g runs rows [b_g, b_{g+1}) of
// partition_by_nnz(a, world) (partition.hpp:55-90) and every product includes
// the band form's exchange over NVLink / NVSwitch:
//
//   windowed (y halo, the north star's form): a band only scatters downward
//     into [lo_g, b_g) (effective_range, partition.hpp:94-102). Boundary rows
//     first; their halo partials go to the owning lower ranks with grouped
//     ncclSend / ncclRecv on a communication stream while the interior rows
//     run; the owners add them (csrc_gpu_halo_accumulate) -- the reference's
//     `effective` accumulation (parallel.hpp:371-382) at GPU granularity.
//   gather (x halo): the band reads x on [lo_g, x_hi_g); with refresh (flags
//     bit 0) only the owned x rows are current, so the rows other bands read go
//     to them (grouped ncclSend / ncclRecv) while the interior rows -- those
//     reading own x only -- run; the boundary rows follow.
//
// Built purely on the public C ABI (band plans, partial products, halo reduce)
// plus NCCL, which is loaded with dlopen so the product library has no link-time
// NCCL dependency (it binds whichever libnccl.so.2 the process already mapped,
// e.g. torch's). ncclCommGetAsyncError is polled by csrc_gpu_band_exec_check and
// after every exchange; an error aborts the communicator and is reported.
// paper_1003_0952_b200/dist.py is the Python (torch.distributed) counterpart;
// both derive the same exchange lists (tests/test_dist.py).
#include <dlfcn.h>
#include <nccl.h>

#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "internal.hpp"

using namespace csrcgpu;

namespace {

struct Nccl {
    void* h = nullptr;
    decltype(&::ncclGetUniqueId) getUniqueId = nullptr;
    decltype(&::ncclCommInitRank) commInitRank = nullptr;
    decltype(&::ncclCommDestroy) commDestroy = nullptr;
    decltype(&::ncclCommAbort) commAbort = nullptr;
    decltype(&::ncclCommGetAsyncError) commGetAsyncError = nullptr;
    decltype(&::ncclGetErrorString) getErrorString = nullptr;
    decltype(&::ncclGroupStart) groupStart = nullptr;
    decltype(&::ncclGroupEnd) groupEnd = nullptr;
    decltype(&::ncclSend) send = nullptr;
    decltype(&::ncclRecv) recv = nullptr;
};

const Nccl& nccl() {
    static Nccl n = [] {
        Nccl v;
        for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
            v.h = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
            if (v.h) break;
        }
        if (!v.h) return v;
        auto sym = [&](const char* s) { return dlsym(v.h, s); };
        v.getUniqueId = reinterpret_cast<decltype(v.getUniqueId)>(sym("ncclGetUniqueId"));
        v.commInitRank = reinterpret_cast<decltype(v.commInitRank)>(sym("ncclCommInitRank"));
        v.commDestroy = reinterpret_cast<decltype(v.commDestroy)>(sym("ncclCommDestroy"));
        v.commAbort = reinterpret_cast<decltype(v.commAbort)>(sym("ncclCommAbort"));
        v.commGetAsyncError = reinterpret_cast<decltype(v.commGetAsyncError)>(sym("ncclCommGetAsyncError"));
        v.getErrorString = reinterpret_cast<decltype(v.getErrorString)>(sym("ncclGetErrorString"));
        v.groupStart = reinterpret_cast<decltype(v.groupStart)>(sym("ncclGroupStart"));
        v.groupEnd = reinterpret_cast<decltype(v.groupEnd)>(sym("ncclGroupEnd"));
        v.send = reinterpret_cast<decltype(v.send)>(sym("ncclSend"));
        v.recv = reinterpret_cast<decltype(v.recv)>(sym("ncclRecv"));
        return v;
    }();
    if (!n.h || !n.commInitRank || !n.send || !n.recv)
        throw Error("band executor: NCCL (libnccl.so.2) is not available in this process");
    return n;
}

#define BX_CUDA(expr)                                                                          \
    do {                                                                                       \
        cudaError_t _e = (expr);                                                               \
        if (_e != cudaSuccess)                                                                 \
            throw Error(std::string("CUDA error: ") + cudaGetErrorString(_e) + " at " + #expr); \
    } while (0)

void nccl_ok(ncclResult_t r, const char* what) {
    if (r != ncclSuccess)
        throw Error(std::string("NCCL error in ") + what + ": " + nccl().getErrorString(r));
}

void abi_ok(int rc) {
    if (rc != 0) throw Error(csrc_gpu_last_error());
}

}  // namespace

struct csrc_gpu_band_exec_s {
    int device = 0;
    int world = 1, rank = 0;
    int form = CSRC_BAND_WINDOWED;
    int dtype = CSRC_DTYPE_F64;
    csrc_gpu_band_lists lists{};
    std::vector<int32_t> send_peer, send_q0, send_q1, recv_peer, recv_q0, recv_q1;
    csrc_gpu_plan_t plan = nullptr;
    ncclComm_t comm = nullptr;
    cudaStream_t comm_stream = nullptr;
    cudaEvent_t ev_ready = nullptr, ev_recv = nullptr;
    int32_t g0 = 0, g1 = 0;  // gather: interior rows (plan-relative)
    void* recv_buf = nullptr; // windowed: received halo partials, concatenated
    std::vector<int64_t> recv_off;
    bool failed = false;
    std::string fail_msg;

    size_t vsize() const { return dtype == CSRC_DTYPE_F32 ? 4 : 8; }
    ncclDataType_t nccl_type() const { return dtype == CSRC_DTYPE_F32 ? ncclFloat : ncclDouble; }

    ~csrc_gpu_band_exec_s() {
        cudaSetDevice(device);
        if (comm_stream) cudaStreamSynchronize(comm_stream);
        if (comm) nccl().commDestroy(comm);
        if (recv_buf) cudaFree(recv_buf);
        if (ev_ready) cudaEventDestroy(ev_ready);
        if (ev_recv) cudaEventDestroy(ev_recv);
        if (comm_stream) cudaStreamDestroy(comm_stream);
        if (plan) csrc_gpu_plan_destroy(plan);
    }

    void poll() {
        if (failed) throw Error(fail_msg);
        ncclResult_t async = ncclSuccess;
        nccl_ok(nccl().commGetAsyncError(comm, &async), "ncclCommGetAsyncError");
        if (async != ncclSuccess && async != ncclInProgress) {
            failed = true;
            fail_msg = std::string("band executor: NCCL communicator failed: ") + nccl().getErrorString(async);
            nccl().commAbort(comm);
            comm = nullptr;
            throw Error(fail_msg);
        }
    }
};

namespace {

// Exchange lists of rank `rank` (the same derivation as paper_1003_0952_b200/dist.py
// halo_plan / gather_plan): windowed -- sends (peer, [q0, q1)) of my halo partials
// [lo, b_g) to their owners, recvs of my rows inside higher ranks' halos; gather --
// x rows I send (mine inside a peer's x range) and receive (a peer's rows inside mine).
void derive_lists(const csrc_host_matrix* a, int world, int rank, int form, csrc_gpu_band_lists& L,
                  std::vector<int32_t>* sp, std::vector<int32_t>* s0, std::vector<int32_t>* s1,
                  std::vector<int32_t>* rp, std::vector<int32_t>* r0, std::vector<int32_t>* r1) {
    std::vector<int32_t> bs(static_cast<size_t>(world) + 1), lo(world), hi(world), xh(world);
    std::vector<int64_t> bn(world);
    abi_ok(csrc_partition_by_nnz(a, world, bs.data(), bn.data()));
    abi_ok(csrc_effective_ranges(a, world, bs.data(), lo.data(), hi.data()));
    L.row_begin = bs[rank];
    L.row_end = bs[rank + 1];
    L.lo = lo[rank];
    auto add = [](std::vector<int32_t>* p, std::vector<int32_t>* q0v, std::vector<int32_t>* q1v, int peer,
                  int32_t q0, int32_t q1) {
        p->push_back(peer);
        q0v->push_back(q0);
        q1v->push_back(q1);
    };
    if (form == CSRC_BAND_WINDOWED) {
        L.x_lo = L.y_lo = lo[rank];
        L.x_hi = bs[rank + 1];
        for (int b = 0; b < rank; ++b) {
            const int32_t q0 = std::max(lo[rank], bs[b]), q1 = std::min(bs[rank], bs[b + 1]);
            if (q0 < q1) add(sp, s0, s1, b, q0, q1);
        }
        for (int c = rank + 1; c < world; ++c) {
            const int32_t q0 = std::max(lo[c], bs[rank]), q1 = std::min(bs[c], bs[rank + 1]);
            if (q0 < q1) add(rp, r0, r1, c, q0, q1);
        }
    } else {
        abi_ok(csrc_bands_x_hi(a, world, bs.data(), xh.data()));
        L.x_lo = lo[rank];
        L.x_hi = xh[rank];
        L.y_lo = bs[rank];
        for (int b = 0; b < world; ++b) {
            if (b == rank) continue;
            int32_t q0 = std::max(lo[rank], bs[b]), q1 = std::min(xh[rank], bs[b + 1]);
            if (q0 < q1) add(rp, r0, r1, b, q0, q1);  // peer b's rows inside my x range
            q0 = std::max(lo[b], bs[rank]);
            q1 = std::min(xh[b], bs[rank + 1]);
            if (q0 < q1) add(sp, s0, s1, b, q0, q1);  // my rows inside peer b's x range
        }
    }
    L.n_sends = static_cast<int32_t>(sp->size());
    L.n_recvs = static_cast<int32_t>(rp->size());
}

template <class F>
void grouped(F&& f) {
    nccl_ok(nccl().groupStart(), "ncclGroupStart");
    try {
        f();
    } catch (...) {
        nccl().groupEnd();
        throw;
    }
    nccl_ok(nccl().groupEnd(), "ncclGroupEnd");
}

}  // namespace

extern "C" {

int csrc_gpu_nccl_get_unique_id(uint8_t* id) {
    return guarded(__func__, [&] {
        if (!id) throw Error("null id");
        ncclUniqueId u;
        nccl_ok(nccl().getUniqueId(&u), "ncclGetUniqueId");
        std::memcpy(id, u.internal, NCCL_UNIQUE_ID_BYTES);
    });
}

int csrc_gpu_band_lists_get(const csrc_host_matrix* a, int32_t world, int32_t rank, int32_t form,
                            csrc_gpu_band_lists* lists, int32_t* send_peer, int32_t* send_q0, int32_t* send_q1,
                            int32_t* recv_peer, int32_t* recv_q0, int32_t* recv_q1) {
    return guarded(__func__, [&] {
        if (!a || !lists) throw Error("null argument");
        if (world < 1 || rank < 0 || rank >= world) throw Error("band lists: need 0 <= rank < world");
        std::vector<int32_t> sp, s0, s1, rp, r0, r1;
        derive_lists(a, world, rank, form, *lists, &sp, &s0, &s1, &rp, &r0, &r1);
        auto out = [](int32_t* dst, const std::vector<int32_t>& v) {
            if (dst) std::copy(v.begin(), v.end(), dst);
        };
        out(send_peer, sp);
        out(send_q0, s0);
        out(send_q1, s1);
        out(recv_peer, rp);
        out(recv_q0, r0);
        out(recv_q1, r1);
    });
}

int csrc_gpu_band_exec_create(const csrc_host_matrix* a, const csrc_gpu_strategy* s, int32_t world, int32_t rank,
                              int32_t form, const uint8_t* id, csrc_gpu_band_exec_t* out) {
    return guarded(__func__, [&] {
        if (!a || !s || !id || !out) throw Error("null argument");
        *out = nullptr;
        if (world < 1 || rank < 0 || rank >= world) throw Error("band executor: need 0 <= rank < world");
        if (form != CSRC_BAND_WINDOWED && form != CSRC_BAND_GATHER) throw Error("band executor: unknown form");
        auto ex = std::make_unique<csrc_gpu_band_exec_s>();
        ex->device = s->device;
        ex->world = world;
        ex->rank = rank;
        ex->form = form;
        ex->dtype = s->dtype;
        BX_CUDA(cudaSetDevice(ex->device));
        derive_lists(a, world, rank, form, ex->lists, &ex->send_peer, &ex->send_q0, &ex->send_q1, &ex->recv_peer,
                     &ex->recv_q0, &ex->recv_q1);
        csrc_gpu_strategy st = *s;
        st.kind = form == CSRC_BAND_WINDOWED ? CSRC_KIND_WINDOWED : CSRC_KIND_GATHER;
        abi_ok(csrc_gpu_plan_create_band(a, &st, ex->lists.row_begin, ex->lists.row_end, &ex->plan));
        csrc_gpu_plan_info info;
        abi_ok(csrc_gpu_plan_get_info(ex->plan, &info));
        if (info.lo != ex->lists.lo || (form == CSRC_BAND_GATHER && info.x_hi != ex->lists.x_hi))
            throw Error("band executor: plan and exchange lists disagree on the band's x range");
        if (form == CSRC_BAND_GATHER) abi_ok(csrc_gpu_gather_interior(ex->plan, &ex->g0, &ex->g1));
        int64_t tot = 0;
        ex->recv_off.push_back(0);
        if (form == CSRC_BAND_WINDOWED)
            for (size_t i = 0; i < ex->recv_q0.size(); ++i) {
                tot += ex->recv_q1[i] - ex->recv_q0[i];
                ex->recv_off.push_back(tot);
            }
        if (tot > 0) BX_CUDA(cudaMalloc(&ex->recv_buf, static_cast<size_t>(tot) * ex->vsize()));
        BX_CUDA(cudaStreamCreateWithFlags(&ex->comm_stream, cudaStreamNonBlocking));
        BX_CUDA(cudaEventCreateWithFlags(&ex->ev_ready, cudaEventDisableTiming));
        BX_CUDA(cudaEventCreateWithFlags(&ex->ev_recv, cudaEventDisableTiming));
        ncclUniqueId u;
        std::memcpy(u.internal, id, NCCL_UNIQUE_ID_BYTES);
        nccl_ok(nccl().commInitRank(&ex->comm, world, u, rank), "ncclCommInitRank");
        *out = ex.release();
    });
}

int csrc_gpu_band_exec_get_info(csrc_gpu_band_exec_t ex, csrc_gpu_band_lists* lists) {
    return guarded(__func__, [&] {
        if (!ex || !lists) throw Error("null argument");
        *lists = ex->lists;
    });
}

int csrc_gpu_band_exec_plan(csrc_gpu_band_exec_t ex, csrc_gpu_plan_t* plan) {
    return guarded(__func__, [&] {
        if (!ex || !plan) throw Error("null argument");
        *plan = ex->plan;
    });
}

int csrc_gpu_band_exec_apply(csrc_gpu_band_exec_t ex, const void* d_x, void* d_y, void* stream, int32_t flags) {
    return guarded(__func__, [&] {
        if (!ex) throw Error("null executor");
        ex->poll();
        BX_CUDA(cudaSetDevice(ex->device));
        cudaStream_t st = static_cast<cudaStream_t>(stream);  // NULL: the legacy default stream
        const csrc_gpu_band_lists& L = ex->lists;
        const size_t E = ex->vsize();
        const ncclDataType_t t = ex->nccl_type();
        if (ex->form == CSRC_BAND_GATHER) {
            const int32_t nrows = L.row_end - L.row_begin;
            const bool refresh = (flags & 1) != 0 && (L.n_sends > 0 || L.n_recvs > 0);
            if (!refresh) {
                abi_ok(csrc_gpu_spmv_device(ex->plan, d_x, d_y, st, 0));
                return;
            }
            // owned x rows are current on `st`; their copies go out while the interior runs
            BX_CUDA(cudaEventRecord(ex->ev_ready, st));
            BX_CUDA(cudaStreamWaitEvent(ex->comm_stream, ex->ev_ready, 0));
            char* xb = static_cast<char*>(const_cast<void*>(d_x));
            grouped([&] {
                for (int i = 0; i < L.n_sends; ++i)
                    nccl_ok(nccl().send(xb + static_cast<size_t>(ex->send_q0[i] - L.x_lo) * E,
                                        static_cast<size_t>(ex->send_q1[i] - ex->send_q0[i]), t, ex->send_peer[i],
                                        ex->comm, ex->comm_stream),
                            "ncclSend");
                for (int i = 0; i < L.n_recvs; ++i)
                    nccl_ok(nccl().recv(xb + static_cast<size_t>(ex->recv_q0[i] - L.x_lo) * E,
                                        static_cast<size_t>(ex->recv_q1[i] - ex->recv_q0[i]), t, ex->recv_peer[i],
                                        ex->comm, ex->comm_stream),
                            "ncclRecv");
            });
            BX_CUDA(cudaEventRecord(ex->ev_recv, ex->comm_stream));
            if (ex->g0 < ex->g1) {
                abi_ok(csrc_gpu_spmv_device_rows(ex->plan, d_x, d_y, st, 0, ex->g0, ex->g1));
                BX_CUDA(cudaStreamWaitEvent(st, ex->ev_recv, 0));
                if (ex->g0 > 0) abi_ok(csrc_gpu_spmv_device_rows(ex->plan, d_x, d_y, st, 0, 0, ex->g0));
                if (ex->g1 < nrows) abi_ok(csrc_gpu_spmv_device_rows(ex->plan, d_x, d_y, st, 0, ex->g1, nrows));
            } else {
                BX_CUDA(cudaStreamWaitEvent(st, ex->ev_recv, 0));
                abi_ok(csrc_gpu_spmv_device(ex->plan, d_x, d_y, st, 0));
            }
        } else if (L.n_sends == 0 && L.n_recvs == 0) {
            abi_ok(csrc_gpu_spmv_device(ex->plan, d_x, d_y, st, 0));  // nothing to exchange (one rank)
        } else {
            // boundary rows (and the y init), then the halo partials travel while the interior runs
            abi_ok(csrc_gpu_spmv_device_part(ex->plan, d_x, d_y, st, 0));
            BX_CUDA(cudaEventRecord(ex->ev_ready, st));
            BX_CUDA(cudaStreamWaitEvent(ex->comm_stream, ex->ev_ready, 0));
            char* yb = static_cast<char*>(d_y);
            char* rb = static_cast<char*>(ex->recv_buf);
            grouped([&] {
                for (int i = 0; i < L.n_sends; ++i)
                    nccl_ok(nccl().send(yb + static_cast<size_t>(ex->send_q0[i] - L.y_lo) * E,
                                        static_cast<size_t>(ex->send_q1[i] - ex->send_q0[i]), t, ex->send_peer[i],
                                        ex->comm, ex->comm_stream),
                            "ncclSend");
                for (int i = 0; i < L.n_recvs; ++i)
                    nccl_ok(nccl().recv(rb + static_cast<size_t>(ex->recv_off[i]) * E,
                                        static_cast<size_t>(ex->recv_q1[i] - ex->recv_q0[i]), t, ex->recv_peer[i],
                                        ex->comm, ex->comm_stream),
                            "ncclRecv");
            });
            BX_CUDA(cudaEventRecord(ex->ev_recv, ex->comm_stream));
            abi_ok(csrc_gpu_spmv_device_part(ex->plan, d_x, d_y, st, 1));  // interior, overlaps the halo
            BX_CUDA(cudaStreamWaitEvent(st, ex->ev_recv, 0));
            for (int i = 0; i < L.n_recvs; ++i)
                abi_ok(csrc_gpu_halo_accumulate(ex->plan, d_y, ex->recv_q0[i] - L.y_lo,
                                                rb + static_cast<size_t>(ex->recv_off[i]) * E,
                                                ex->recv_q1[i] - ex->recv_q0[i], st));
        }
        ex->poll();
    });
}

int csrc_gpu_band_exec_check(csrc_gpu_band_exec_t ex) {
    return guarded(__func__, [&] {
        if (!ex) throw Error("null executor");
        ex->poll();
    });
}

void csrc_gpu_band_exec_destroy(csrc_gpu_band_exec_t ex) { delete ex; }

}  // extern "C"

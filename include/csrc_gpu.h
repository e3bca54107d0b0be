/*
 * csrc_gpu.h — C-ABI drop-in boundary of the B200-native CSRC SpMV.
 *
 * The reference (arXiv 1003.0952 artefact, header-only C++ under
 * /root/reference/proj/include/csrc) exposes its hot path as C++ calls:
 *
 *   Vector spmv_csrc(const CsrcMatrix&, const Vector&)        kernels.hpp:25-43
 *   Vector spmv_csrc_transpose(const CsrcMatrix&, const Vector&) kernels.hpp:47-65
 *   ParallelSpmv(const CsrcMatrix&, Strategy)                  parallel.hpp:153-156
 *   ParallelSpmv(const CsrcMatrix&, Strategy, LocalBuffersPlan) parallel.hpp:158-161
 *   ParallelSpmv(const CsrcMatrix&, Strategy, ColorfulPlan)    parallel.hpp:163-166
 *   Vector ParallelSpmv::apply(const Vector&)                  parallel.hpp:183-187
 *   void   ParallelSpmv::apply(const Vector& x, Vector& y)     parallel.hpp:189-220
 *   const PhaseTimings& ParallelSpmv::last_timings()           parallel.hpp:222
 *   int    ParallelSpmv::buffers_allocated()                   parallel.hpp:223
 *   RowPartition partition_by_nnz(const CsrcMatrix&, int p)    partition.hpp:55-90
 *   std::vector<EffectiveRange> effective_ranges(...)          partition.hpp:104-109
 *   IntervalPlan build_interval_plan(...)                      partition.hpp:113-134
 *   Coloring color_rows(build_conflict_graph(a, mode), order)  coloring.hpp:93-164
 *   ColoringValidity validate_coloring(const CsrcMatrix&, const Coloring&) coloring.hpp:175-198
 *   double working_set_kb(n, nnz_stored, value_symmetric)      working_set.hpp:17-25
 *
 * Every entry point below replaces one of those; the reference has no FFI of
 * its own, so the C++ wrapper include/csrc_gpu.hpp restores the exact C++
 * call shapes on top of this ABI.
 *
 * Conventions
 *  - Plain pointers and sizes only; no C++ or torch types cross the boundary.
 *  - Return 0 on success, nonzero on error; csrc_gpu_last_error() returns a
 *    thread-local message with the reference's wording where one exists
 *    (e.g. "spmv_csrc: x has length 3, expected 4").
 *  - A plan copies the matrix to the device; the host matrix may be freed
 *    after csrc_gpu_plan_create returns. One apply in flight per plan.
 *  - Indices are int32 (csrc::index_t, common.hpp:10); counts int64
 *    (csrc::count_t, common.hpp:11); values f64 (csrc::Vector, common.hpp:20)
 *    or f32 for CSRC_DTYPE_F32 plans (host vectors stay f64 at the boundary).
 */
#ifndef CSRC_GPU_H
#define CSRC_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CSRC_GPU_ABI_VERSION 1

/* ------------------------------------------------------------------ types */

/* Borrowed view of a csrc::CsrcMatrix (csrc_matrix.hpp:14-30). */
typedef struct {
    int32_t n;                 /* rows = cols                                  */
    int64_t k;                 /* stored off-diagonal pairs = ia[n]            */
    const double* ad;          /* diagonal, length n                           */
    const int32_t* ia;         /* row pointers into ja/al/au, length n+1       */
    const int32_t* ja;         /* lower column indices, ja[t] < row(t)         */
    const double* al;          /* lower values a_ij, length k                  */
    const double* au;          /* upper values a_ji, length k; NULL iff value_symmetric */
    int32_t value_symmetric;   /* 1: au elided, al serves both (csrc_matrix.hpp:29) */
} csrc_host_matrix;

/* Strategy kinds. SEQUENTIAL / LOCAL_BUFFERS / COLORFUL mirror
 * csrc::StrategyKind (parallel.hpp:16); ATOMIC and WINDOWED are the GPU-only
 * kernels the north star asks for; GATHER is the fastest. */
enum {
    CSRC_KIND_SEQUENTIAL = 0,   /* no buffers: the gather kernel (windowed for band plans) */
    CSRC_KIND_LOCAL_BUFFERS = 1,/* windowed kernel into private band buffers + accumulation pass */
    CSRC_KIND_COLORFUL = 2,     /* conflict-free row classes in class order, no atomics (one wavefront launch) */
    CSRC_KIND_ATOMIC = 3,       /* global fp64/fp32 red.global scatter baseline */
    CSRC_KIND_WINDOWED = 4,     /* TMA tiles, smem y rings, red.global flush (CSRC model bytes) */
    CSRC_KIND_GATHER = 5        /* transposed gather: the plan lays out each row's lower pairs and
                                   the pairs naming it as column as one entry stream (+4 B/pair
                                   over the CSRC model), no scatter, bit-reproducible */
};

/* csrc::AccumMethod (parallel.hpp:17) */
enum {
    CSRC_ACCUM_ALL_IN_ONE = 0,
    CSRC_ACCUM_PER_BUFFER = 1,
    CSRC_ACCUM_EFFECTIVE = 2,
    CSRC_ACCUM_INTERVAL = 3
};

/* csrc::ConflictMode (coloring.hpp:15-18) and csrc::ColorOrder (coloring.hpp:35) */
enum { CSRC_CONFLICT_NEIGHBORHOOD = 0, CSRC_CONFLICT_EXACT = 1 };
enum { CSRC_ORDER_NATURAL = 0, CSRC_ORDER_LARGEST_FIRST = 1, CSRC_ORDER_SMALLEST_LAST = 2 };

enum { CSRC_DTYPE_F64 = 0, CSRC_DTYPE_F32 = 1 };

/* Superset of csrc::Strategy {kind, accum, p} (parallel.hpp:19-23). */
typedef struct {
    int32_t kind;           /* CSRC_KIND_*                                          */
    int32_t accum;          /* CSRC_ACCUM_* (local buffers only)                    */
    int32_t p;              /* reference thread count; >= 1 (validated like parallel.hpp:231-233).
                               The device chooses its own band count; p is kept for the
                               reference's error behaviour and allocation_stats.        */
    int32_t dtype;          /* CSRC_DTYPE_*                                         */
    int32_t conflict_mode;  /* CSRC_CONFLICT_* (colorful only)                      */
    int32_t color_order;    /* CSRC_ORDER_*    (colorful only)                      */
    int32_t device;         /* CUDA device ordinal                                  */
    int32_t bands;          /* device bands (CTAs) for windowed/local-buffers; 0 = auto */
} csrc_gpu_strategy;

/* csrc::PhaseTimings (parallel.hpp:26-30), milliseconds, from CUDA events on
 * the plan's stream; halo_ms is the multi-GPU reduce (0 on one device). */
typedef struct {
    double init_ms;
    double compute_ms;
    double accumulate_ms;
    double halo_ms;
} csrc_gpu_timings;

typedef struct {
    int32_t n;
    int64_t k;
    int32_t kind;
    int32_t dtype;
    int32_t bands;              /* device bands (CTA count) used                  */
    int32_t buffers_allocated;  /* csrc::ParallelSpmv::buffers_allocated (parallel.hpp:223) */
    int32_t n_colors;           /* colorful only                                  */
    int32_t row_begin, row_end; /* rows owned by this plan (band plans)           */
    int32_t lo;                 /* effective_range lo of the owned rows           */
    int64_t model_bytes;        /* working_set model bytes (working_set.hpp:17-25) */
    int64_t device_bytes;       /* device memory held by the plan                 */
    int32_t n_windows;          /* windowed: scatter-distance windows             */
    int32_t win_lo[6], win_hi[6]; /* windowed: distance interval of each window   */
    int32_t lanes;              /* windowed / gather: lanes per row               */
    int32_t stages;             /* windowed: TMA pipeline depth; gather: buffers  */
    int32_t smem_bytes;         /* windowed / gather: dynamic shared memory per CTA */
    int32_t launches_per_apply; /* kernels launched per product                   */
    double  captured_fraction;  /* windowed: pairs whose scatter lands in a window */
    int64_t stream_bytes;       /* bytes one product moves in the plan's device layout
                                   (= model_bytes for the CSRC kernels; gather: its entry
                                   stream)                          */
    int32_t row_patterns;       /* gather: column-offset patterns (0 = explicit indices) */
    int32_t x_hi;               /* x is read on [lo, x_hi): row_end for the scatter kernels;
                                   gather band plans also read x above the band       */
    int32_t m_cols;             /* rectangular plans: columns of A (x length); 0 = square */
    int64_t rect_nnz;           /* rectangular plans: entries of the CSR tail        */
    int32_t gather_form;        /* gather plans: 1 k_gather_rows, 2 k_gather_staged,
                                   3 k_gather_sell; 0 for the other kinds            */
    int32_t csr_cols;           /* CSR plans: columns of A (x length); 0 otherwise  */
} csrc_gpu_plan_info;

typedef struct csrc_gpu_plan_s* csrc_gpu_plan_t;

/* -------------------------------------------------------------- errors */

const char* csrc_gpu_last_error(void);
int csrc_gpu_abi_version(void);
int csrc_gpu_device_count(void);

/* ---------------------------------------------------------------- plans */

/* ParallelSpmv(const CsrcMatrix&, Strategy) (parallel.hpp:153-156). */
int csrc_gpu_plan_create(const csrc_host_matrix* a, const csrc_gpu_strategy* s,
                         csrc_gpu_plan_t* out);

/* ParallelSpmv(a, s, ColorfulPlan) (parallel.hpp:163-166): explicit coloring.
 * The coloring is validated with the exact write-set check of
 * validate_coloring (coloring.hpp:175-198); an invalid one is rejected with
 * "coloring violation: rows A and B both write y[Q]". */
int csrc_gpu_plan_create_colored(const csrc_host_matrix* a, const csrc_gpu_strategy* s,
                                 const int32_t* color, int32_t n_colors,
                                 csrc_gpu_plan_t* out);

/* ParallelSpmv(a, s, LocalBuffersPlan) (parallel.hpp:158-161): explicit
 * contiguous band partition block_start[0..bands] (0 .. n). */
int csrc_gpu_plan_create_partitioned(const csrc_host_matrix* a, const csrc_gpu_strategy* s,
                                     const int32_t* block_start, int32_t bands,
                                     csrc_gpu_plan_t* out);

/* Multi-GPU band plan: rows [row_begin, row_end) of a; x and y device
 * vectors passed to the apply calls cover [lo, row_end) where lo is the
 * band's effective_range lo (partition.hpp:94-102): y[0 .. row_begin-lo) is
 * the halo partial owed to lower bands, y[row_begin-lo ..) the owned rows
 * (still missing the halo partials of higher bands). */
int csrc_gpu_plan_create_band(const csrc_host_matrix* a, const csrc_gpu_strategy* s,
                              int32_t row_begin, int32_t row_end, csrc_gpu_plan_t* out);

/* spmv_csr (kernels.hpp:7-22) on the GPU: a plan over a general CSR matrix
 * (n_rows x n_cols, any pattern, csr.hpp:28-51), run by the gather kernels on
 * the rows as they stand; strategy kind SEQUENTIAL or GATHER. x has n_cols
 * entries, y n_rows; no transpose product. The reference's Format::csr
 * baseline of the CSRC-vs-CSR comparison (bench.hpp:203-215). */
int csrc_gpu_plan_create_csr(int32_t n_rows, int32_t n_cols, const int32_t* row_ptr, const int32_t* col_idx,
                             const double* values, const csrc_gpu_strategy* s, csrc_gpu_plan_t* out);

/* ParallelSpmv(const CsrcRectMatrix&, Strategy) (parallel.hpp:168-181) and
 * spmv_csrc_rect (kernels.hpp:69-91): the n x n CSRC part `a` plus the CSR
 * tail over columns n..m_cols-1 (tail_row_ptr[n+1], local column indices,
 * csrc_matrix.hpp:35-39). x has m_cols entries; every kernel kind runs its
 * square product, then one tail pass adds the row sums of the tail. No
 * transpose product and no band plans for rectangular matrices. */
int csrc_gpu_plan_create_rect(const csrc_host_matrix* a, const csrc_gpu_strategy* s, int32_t m_cols,
                              const int32_t* tail_row_ptr, const int32_t* tail_col_idx,
                              const double* tail_values, csrc_gpu_plan_t* out);

/* ParallelSpmv(const CsrcRectMatrix&, Strategy, ColorfulPlan | LocalBuffersPlan)
 * (parallel.hpp:173-181): a rectangular plan with an explicit colouring
 * (color[n], n_colors; block_start NULL) or band partition (block_start[bands+1];
 * color NULL). */
int csrc_gpu_plan_create_rect_plan(const csrc_host_matrix* a, const csrc_gpu_strategy* s, int32_t m_cols,
                                   const int32_t* tail_row_ptr, const int32_t* tail_col_idx,
                                   const double* tail_values, const int32_t* color, int32_t n_colors,
                                   const int32_t* block_start, int32_t bands, csrc_gpu_plan_t* out);

/* ParallelSpmv::colorful_plan (parallel.hpp:226): the colouring a colorful plan
 * runs (color[n] may be NULL to query *n_colors; 0 for other kinds). */
int csrc_gpu_plan_get_coloring(csrc_gpu_plan_t plan, int32_t* color, int32_t* n_colors);

void csrc_gpu_plan_destroy(csrc_gpu_plan_t plan);
int csrc_gpu_plan_get_info(csrc_gpu_plan_t plan, csrc_gpu_plan_info* info);

/* ----------------------------------------------------------- products */

/* Drop-in: x_host length n (f64), y_host length n (f64), host memory.
 * H2D of x, the product, D2H of y; returns after y is on the host.
 * ParallelSpmv::apply(x, y) (parallel.hpp:189-220) / spmv_csrc (kernels.hpp:25). */
int csrc_gpu_spmv(csrc_gpu_plan_t plan, const double* x_host, int64_t x_len, double* y_host);

/* One-shot spmv_csrc / spmv_csrc_transpose (kernels.hpp:25-65) of a host matrix,
 * no plan: the CSRC arrays stream to the device as stored, row chunk by row chunk
 * (pinned double-buffered staging, copies overlapped with the global-atomic kernel
 * on the previous chunk); x, y host vectors of length n. For a single product the
 * plan-free path wins: a plan's preprocessing costs seconds at C5. */
int csrc_gpu_spmv_oneshot(const csrc_host_matrix* a, const double* x_host, int64_t x_len, double* y_host,
                          int32_t transpose, int32_t device);

/* spmv_csrc_transpose (kernels.hpp:47-65): al/au swapped, zero-copy. */
int csrc_gpu_spmv_transpose(csrc_gpu_plan_t plan, const double* x_host, int64_t x_len,
                            double* y_host);

/* Throughput form: device pointers in the plan's dtype, enqueued on `stream`
 * (a cudaStream_t; NULL = the plan's own stream). Asynchronous.
 * flags bit 0: transpose. */
int csrc_gpu_spmv_device(csrc_gpu_plan_t plan, const void* d_x, void* d_y, void* stream,
                         int32_t flags);

/* Same product replayed through a CUDA graph captured on first use for the
 * given (d_x, d_y, stream) triple. */
int csrc_gpu_spmv_device_graph(csrc_gpu_plan_t plan, const void* d_x, void* d_y,
                               void* stream);

/* Multi-GPU halo reduce: y_owned[dst_off + i] += recv[i] for i < len, on
 * `stream`; both device pointers in the plan's dtype. */
int csrc_gpu_halo_accumulate(csrc_gpu_plan_t plan, void* d_y, int64_t dst_off,
                             const void* d_recv, int64_t len, void* stream);

/* Rows of the band whose scatters reach below row_begin (must finish before
 * the halo can be shipped); the rest is interior work. */
int csrc_gpu_band_split(csrc_gpu_plan_t plan, int32_t* boundary_rows_end);

/* Partial products for overlap: rows [row_begin, split) or [split, row_end)
 * of a band plan; part = 0 boundary, 1 interior. The y init is done by
 * part 0 (zero [lo, row_end)). */
int csrc_gpu_spmv_device_part(csrc_gpu_plan_t plan, const void* d_x, void* d_y, void* stream,
                              int32_t part);

/* Gather plans: rows [*rows_begin, *rows_end) (relative to the plan's rows,
 * 256-aligned inward) read x only on the plan's own rows -- for band plans
 * they can run while an x-halo exchange is in flight (paper_1003_0952_b200.dist). */
int csrc_gpu_gather_interior(csrc_gpu_plan_t plan, int32_t* rows_begin, int32_t* rows_end);

/* Gather plans: the product restricted to rows [rows_begin, rows_end) (plan-relative;
 * begin a multiple of 256, end a multiple of 256 or the last row); d_x / d_y as for
 * csrc_gpu_spmv_device, only the range's y rows are written. flags bit 0: transpose. */
int csrc_gpu_spmv_device_rows(csrc_gpu_plan_t plan, const void* d_x, void* d_y, void* stream, int32_t flags,
                              int32_t rows_begin, int32_t rows_end);

/* csrc::ParallelSpmv::last_timings (parallel.hpp:222); synchronises on the
 * last apply's events. Timing events are recorded only when enabled. */
int csrc_gpu_set_timing(csrc_gpu_plan_t plan, int32_t enabled);
int csrc_gpu_last_timings(csrc_gpu_plan_t plan, csrc_gpu_timings* t);

/* Kernel-only timing helper for benchmarks: runs `reps` products back to
 * back on the plan's stream (device pointers) and writes the per-product
 * CUDA-event durations (ms) of the compute kernel(s) into ms_out[reps]. If
 * flush_bytes > 0 an L2-flush write of that many bytes runs before every
 * product, outside the timed interval. */
int csrc_gpu_time_products(csrc_gpu_plan_t plan, const void* d_x, void* d_y, int32_t reps,
                           int64_t flush_bytes, double* ms_out, double* kernel_ms_out);

/* Same, with x given on the host: x is uploaded once into the plan's own
 * device vectors (converted to the plan's dtype), then `reps` device-resident
 * products are timed. For harnesses without device memory of their own
 * (the csrc_bench CLI). */
int csrc_gpu_time_products_host(csrc_gpu_plan_t plan, const double* x_host, int64_t x_len, int32_t reps,
                                int64_t flush_bytes, double* ms_out, double* kernel_ms_out);

/* ------------------------------------------------- host plan builders
 * Product-side, scalable re-implementations of the reference's plan
 * functions; bit-exact with them (tests/test_plans.py). */

/* partition_by_nnz (partition.hpp:55-90): block_start[p+1], block_nnz[p]. */
int csrc_partition_by_nnz(const csrc_host_matrix* a, int32_t p, int32_t* block_start,
                          int64_t* block_nnz);

/* effective_ranges (partition.hpp:94-109): lo[p], hi[p] (inclusive). */
int csrc_effective_ranges(const csrc_host_matrix* a, int32_t p, const int32_t* block_start,
                          int32_t* lo, int32_t* hi);

/* Multi-GPU gather bands: x_hi[b] = one past the last row that reads x in band b
 * (rows naming one of band b's rows as a lower column), at least block_start[b+1];
 * band b reads x on [effective_range lo, x_hi[b]) (paper_1003_0952_b200.dist). */
int csrc_bands_x_hi(const csrc_host_matrix* a, int32_t p, const int32_t* block_start, int32_t* x_hi);

/* build_interval_plan (partition.hpp:113-134). Two-call protocol: pass NULL
 * outputs to get the sizes, then buffers of those sizes.
 * iv_begin/iv_end[n_intervals], contrib_ptr[n_intervals+1], contrib[n_contrib],
 * boundaries[n_boundaries]. */
int csrc_interval_plan(int32_t p, const int32_t* lo, const int32_t* hi, int32_t* n_intervals,
                       int32_t* n_contrib, int32_t* n_boundaries, int32_t* iv_begin,
                       int32_t* iv_end, int32_t* contrib_ptr, int32_t* contrib,
                       int32_t* boundaries);

/* color_rows(build_conflict_graph(a, mode), order) (coloring.hpp:93-164):
 * color[n], *n_colors. CSR adjacency, no std::set; identical first-fit result. */
int csrc_color_rows(const csrc_host_matrix* a, int32_t mode, int32_t order, int32_t* color,
                    int32_t* n_colors);

/* Conflict-graph edge counts (direct, indirect) of build_conflict_graph. */
int csrc_conflict_edge_counts(const csrc_host_matrix* a, int32_t mode, int64_t* n_direct,
                              int64_t* n_indirect);

/* validate_coloring (coloring.hpp:175-198): returns 0 and sets *valid; on a
 * violation row_a, row_b, position describe the first violating pair. */
int csrc_validate_coloring(const csrc_host_matrix* a, const int32_t* color, int32_t n_colors,
                           int32_t* valid, int32_t* row_a, int32_t* row_b, int32_t* position);

/* ColorfulPlan::slice (parallel.hpp:69-93): slices[n_colors * p * 2]
 * (start, end) per class per worker. */
int csrc_colorful_slices(const csrc_host_matrix* a, const int32_t* color, int32_t n_colors,
                         int32_t p, int64_t* slices);

/* working_set_kb (working_set.hpp:17-25) in bytes, and count_ops flops
 * (cost_model.hpp:20-42, Format::csrc / csrc_sym). */
int64_t csrc_model_bytes(int64_t n, int64_t nnz_stored, int32_t value_symmetric, int32_t dtype);
int64_t csrc_model_flops(int64_t n, int64_t nnz_full);

/* ------------------------------------------------ multi-GPU band executor
 * One per rank (one process per GPU). Rank g owns rows [b_g, b_{g+1}) of
 * partition_by_nnz(a, world) (partition.hpp:55-90); every product includes the
 * band form's exchange over NCCL (grouped ncclSend / ncclRecv on the executor's
 * communication stream, overlapped with interior rows):
 *   CSRC_BAND_WINDOWED  y halo: boundary rows' partials for [lo_g, b_g)
 *                       (effective_range, partition.hpp:94-102) go to their
 *                       owners, which add them -- the `effective` accumulation
 *                       (parallel.hpp:371-382) at GPU granularity;
 *   CSRC_BAND_GATHER    x halo (flags bit 0 = refresh): the owned x rows other
 *                       bands read go to them before the boundary rows run.
 * Device vectors: x covers [x_lo, x_hi), y covers [y_lo, row_end) (the lists).
 * NCCL is loaded at run time (libnccl.so.2); the communicator's async errors
 * are polled around every product and by csrc_gpu_band_exec_check. */
enum { CSRC_BAND_WINDOWED = 0, CSRC_BAND_GATHER = 1 };

typedef struct {
    int32_t row_begin, row_end; /* owned rows                                   */
    int32_t lo;                 /* effective_range lo of the owned rows          */
    int32_t x_lo, x_hi;         /* the band's x range                            */
    int32_t y_lo;               /* the band's y vector starts here               */
    int32_t n_sends, n_recvs;   /* exchange messages per product                 */
} csrc_gpu_band_lists;

typedef struct csrc_gpu_band_exec_s* csrc_gpu_band_exec_t;

/* ncclGetUniqueId on one rank (id: 128 bytes); the caller broadcasts it. */
int csrc_gpu_nccl_get_unique_id(uint8_t* id);

/* The exchange lists of rank `rank` (host only, no NCCL): sizes in *lists;
 * arrays of n_sends / n_recvs entries (peer, [q0, q1) global rows), or NULL. */
int csrc_gpu_band_lists_get(const csrc_host_matrix* a, int32_t world, int32_t rank, int32_t form,
                            csrc_gpu_band_lists* lists, int32_t* send_peer, int32_t* send_q0, int32_t* send_q1,
                            int32_t* recv_peer, int32_t* recv_q0, int32_t* recv_q1);

int csrc_gpu_band_exec_create(const csrc_host_matrix* a, const csrc_gpu_strategy* s, int32_t world, int32_t rank,
                              int32_t form, const uint8_t* nccl_id, csrc_gpu_band_exec_t* out);
int csrc_gpu_band_exec_get_info(csrc_gpu_band_exec_t ex, csrc_gpu_band_lists* lists);
/* the band plan the executor runs (owned by the executor) */
int csrc_gpu_band_exec_plan(csrc_gpu_band_exec_t ex, csrc_gpu_plan_t* plan);
/* y = A x on the band, exchange included, enqueued on `stream` (NULL: legacy stream). */
int csrc_gpu_band_exec_apply(csrc_gpu_band_exec_t ex, const void* d_x, void* d_y, void* stream, int32_t flags);
/* ncclCommGetAsyncError: nonzero (and the communicator aborted) after a failure. */
int csrc_gpu_band_exec_check(csrc_gpu_band_exec_t ex);
void csrc_gpu_band_exec_destroy(csrc_gpu_band_exec_t ex);

/* ------------------------------------------------ CSRC construction
 * Device re-implementations of the reference's construction pipeline
 * (paper_1003_0952_b200/csrc/assemble.cu). Results are host arrays owned by
 * the returned handle, bit-exact with the reference (tests/test_gpu_assemble.py):
 * values are copies of input values, duplicates summed in input order. */
typedef struct csrc_built_s* csrc_built_t;

/* build_csr (csr.hpp:55-92): canonical CSR from m triplets (rows[e], cols[e],
 * vals[e]); duplicates summed; "build_csr: entry (r, c) outside RxC bounds"
 * names the first out-of-bounds triplet in input order. */
int csrc_gpu_build_csr(int32_t n_rows, int32_t n_cols, int64_t m, const int32_t* rows,
                       const int32_t* cols, const double* vals, int32_t device, csrc_built_t* out);

/* csr_to_csrc(build_csr(t)) (csrc_matrix.hpp:44-91) without the host round
 * trip: "csr_to_csrc: entry (i, j) has no transpose (j, i)" / "row i has no
 * diagonal entry" report the first failure in the reference's row-major order;
 * value_symmetric set (and au dropped) iff every pair matches exactly. */
int csrc_gpu_build_csrc(int32_t n, int64_t m, const int32_t* rows, const int32_t* cols,
                        const double* vals, int32_t device, csrc_built_t* out);

/* csr_to_csrc (csrc_matrix.hpp:44-91) of a canonical CSR. */
int csrc_gpu_csr_to_csrc(int32_t n_rows, int32_t n_cols, const int32_t* row_ptr,
                         const int32_t* col_idx, const double* values, int32_t device,
                         csrc_built_t* out);

/* decompose_rect (csrc_matrix.hpp:113-142, symmetrize = false): CSRC square
 * part + CSR tail over columns n..m-1 (local indices). */
int csrc_gpu_decompose_rect(int32_t n_rows, int32_t n_cols, const int32_t* row_ptr,
                            const int32_t* col_idx, const double* values, int32_t device,
                            csrc_built_t* out);

/* Views into a handle (valid until csrc_built_free). */
int csrc_built_matrix(csrc_built_t b, csrc_host_matrix* m);
int csrc_built_csr(csrc_built_t b, int32_t* n_rows, int32_t* n_cols, int64_t* nnz,
                   const int32_t** row_ptr, const int32_t** col_idx, const double** values);
int csrc_built_rect_tail(csrc_built_t b, int32_t* m_cols, int64_t* nnz, const int32_t** row_ptr,
                         const int32_t** col_idx, const double** values);
/* wall-clock ms of the phases: [0] H2D, [1] sort + reduce, [2] CSR -> CSRC, [3] D2H */
int csrc_built_timings(csrc_built_t b, double* ms4);
void csrc_built_free(csrc_built_t b);

/* --------------------------------------------------------- fixtures
 * Deterministic synthetic FE matrices for the BASELINE configs, assembled
 * directly in CSRC form. */
enum {
    CSRC_MESH_GRID2D_Q1 = 0,    /* 9-point, nx*ny nodes                       */
    CSRC_MESH_GRID3D_27 = 1,    /* 27-point, nx*ny*nz nodes                   */
    CSRC_MESH_ELASTICITY = 2,   /* 27-point nodes x 3 dof, 3x3 blocks         */
    CSRC_MESH_GRID3D_27_RCM = 3 /* 27-point, random permutation + RCM         */
};

typedef struct {
    int32_t mesh;       /* CSRC_MESH_*           */
    int32_t nx, ny, nz; /* nodes per axis (nz=1 for 2D) */
    uint64_t seed;      /* value / permutation seed */
    double diag_base;   /* diagonal = diag_base + U(0,1) */
    int32_t threads;    /* host threads, 0 = all */
} csrc_fixture_spec;

typedef struct csrc_fixture_s* csrc_fixture_t;

int csrc_fixture_generate(const csrc_fixture_spec* spec, csrc_fixture_t* out);
int csrc_fixture_matrix(csrc_fixture_t fx, csrc_host_matrix* m);
/* x ~ U(-1,1) from the fixture seed. */
const double* csrc_fixture_x(csrc_fixture_t fx);
/* final-ordering index of natural node/dof u (identity unless RCM). */
const int32_t* csrc_fixture_order(csrc_fixture_t fx);
void csrc_fixture_free(csrc_fixture_t fx);

/* Fixture hash: U01(seed, a, b) in [0,1). Exposed so the
 * oracle-side triplet generator can be cross-checked. */
double csrc_fixture_u01(uint64_t seed, uint64_t a, uint64_t b);

#ifdef __cplusplus
}
#endif

#endif /* CSRC_GPU_H */

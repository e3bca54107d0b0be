/*
 * ORACLE — TEST INFRASTRUCTURE ONLY. Never linked into, or called by, the
 * product (paper_1003_0952_b200/). Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load it, and only as
 * the checker or the CPU baseline.
 *
 * Plain-C restatement of the reference algorithms on the CSRC hot path
 * (/root/reference/proj/include/csrc/...). Each function cites the file:line
 * it follows. Parity is pinned: tests/test_oracle.py checks every function
 * against the reference's own known answers (tests/golden/known_answers.json)
 * and against the reference compiled from its headers (oracle/_ref, golden
 * vectors in tests/golden/*.npz made by tests/golden/make_golden.py).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef int32_t index_t;  /* common.hpp:10 */
typedef int64_t count_t;  /* common.hpp:11 */

/* ------------------------------------------------------------------ SpMV */

/* spmv_csrc, kernels.hpp:25-43. Exact reference FP order: y[i] = ad*xi + sum
 * of al*x[j] in ascending t, then transposed contributions from later rows
 * arrive in ascending row order. au == NULL means value-symmetric (upper()
 * returns al, csrc_matrix.hpp:29). */
void oracle_spmv_csrc(index_t n, const double* ad, const index_t* ia, const index_t* ja,
                      const double* al, const double* au, const double* x, double* y) {
    const double* up = au ? au : al;
    for (index_t i = 0; i < n; ++i) y[i] = 0.0;
    for (index_t i = 0; i < n; ++i) {
        const double xi = x[i];
        double yi = ad[i] * xi;
        for (index_t t = ia[i]; t < ia[i + 1]; ++t) {
            const index_t j = ja[t];
            yi += al[t] * x[j];
            y[j] += up[t] * xi;
        }
        y[i] = yi;
    }
}

/* spmv_csrc_rect, kernels.hpp:69-91: per row the square CSRC updates, then
 * the CSR tail over x[n + tcol] (x has length m). */
void oracle_spmv_csrc_rect(index_t n, const double* ad, const index_t* ia, const index_t* ja,
                           const double* al, const double* au, const index_t* trp,
                           const index_t* tci, const double* tva, const double* x, double* y) {
    const double* up = au ? au : al;
    memset(y, 0, sizeof(double) * (size_t)n);
    for (index_t i = 0; i < n; ++i) {
        const double xi = x[i];
        double yi = ad[i] * xi;
        for (index_t t = ia[i]; t < ia[i + 1]; ++t) {
            const index_t j = ja[t];
            yi += al[t] * x[j];
            y[j] += up[t] * xi;
        }
        for (index_t q = trp[i]; q < trp[i + 1]; ++q) yi += tva[q] * x[n + tci[q]];
        y[i] = yi;
    }
}

/* spmv_csrc_transpose, kernels.hpp:47-65: al and au swap roles. */
void oracle_spmv_csrc_transpose(index_t n, const double* ad, const index_t* ia,
                                const index_t* ja, const double* al, const double* au,
                                const double* x, double* y) {
    if (!au) {
        oracle_spmv_csrc(n, ad, ia, ja, al, NULL, x, y);
        return;
    }
    oracle_spmv_csrc(n, ad, ia, ja, au, al, x, y);
}

/* compute_block + buffers (parallel.hpp:286-307, 359-395, accumulation in
 * ascending buffer id) for a given partition; the reference's local-buffers
 * result with the `effective` reduction order. Scratch: p*n doubles. */
void oracle_spmv_local_buffers(index_t n, const double* ad, const index_t* ia,
                               const index_t* ja, const double* al, const double* au,
                               const double* x, int p, const index_t* block_start, double* y,
                               double* scratch) {
    const double* up = au ? au : al;
    memset(scratch, 0, sizeof(double) * (size_t)p * (size_t)n);
    for (int w = 0; w < p; ++w) {
        double* buf = scratch + (size_t)w * (size_t)n;
        for (index_t i = block_start[w]; i < block_start[w + 1]; ++i) {
            const double xi = x[i];
            double yi = ad[i] * xi;
            for (index_t t = ia[i]; t < ia[i + 1]; ++t) {
                const index_t j = ja[t];
                yi += al[t] * x[j];
                buf[j] += up[t] * xi;
            }
            buf[i] = yi;
        }
    }
    for (index_t q = 0; q < n; ++q) {
        double s = scratch[q];
        for (int b = 1; b < p; ++b) s += scratch[(size_t)b * n + q];
        y[q] = s;
    }
}

/* ---------------------------------------------------------- construction */

typedef struct {
    index_t row, col;
    double val;
    count_t order;
} trip_t;

static int trip_cmp(const void* a, const void* b) {
    const trip_t* x = (const trip_t*)a;
    const trip_t* y = (const trip_t*)b;
    if (x->row != y->row) return x->row < y->row ? -1 : 1;
    if (x->col != y->col) return x->col < y->col ? -1 : 1;
    if (x->order != y->order) return x->order < y->order ? -1 : 1;
    return 0;
}

/* build_csr, csr.hpp:55-92: bounds check, sort by (row, col), sum duplicates
 * (in input order among equal keys), row pointers. Returns 0, or 1 on an
 * out-of-bounds entry (*bad = its index). Outputs sized by the caller
 * (row_ptr n+1, col/val m). *nnz = stored entries. */
int oracle_build_csr(index_t n_rows, index_t n_cols, count_t m, const index_t* rows,
                     const index_t* cols, const double* vals, index_t* row_ptr,
                     index_t* col_idx, double* values, count_t* nnz, count_t* bad) {
    for (count_t e = 0; e < m; ++e) {
        if (rows[e] < 0 || rows[e] >= n_rows || cols[e] < 0 || cols[e] >= n_cols) {
            *bad = e;
            return 1;
        }
    }
    trip_t* t = (trip_t*)malloc(sizeof(trip_t) * (size_t)(m > 0 ? m : 1));
    for (count_t e = 0; e < m; ++e) {
        t[e].row = rows[e];
        t[e].col = cols[e];
        t[e].val = vals[e];
        t[e].order = e;
    }
    qsort(t, (size_t)m, sizeof(trip_t), trip_cmp);
    for (index_t i = 0; i <= n_rows; ++i) row_ptr[i] = 0;
    count_t k = 0;
    for (count_t e = 0; e < m; ++e) {
        if (e > 0 && t[e - 1].row == t[e].row && t[e - 1].col == t[e].col) {
            values[k - 1] += t[e].val;
            continue;
        }
        col_idx[k] = t[e].col;
        values[k] = t[e].val;
        ++k;
        ++row_ptr[t[e].row + 1];
    }
    for (index_t i = 0; i < n_rows; ++i) row_ptr[i + 1] += row_ptr[i];
    *nnz = k;
    free(t);
    return 0;
}

static int csr_find(const index_t* row_ptr, const index_t* col_idx, index_t r, index_t c,
                    count_t* pos) {
    index_t lo = row_ptr[r], hi = row_ptr[r + 1];
    while (lo < hi) {
        index_t mid = lo + (hi - lo) / 2;
        if (col_idx[mid] < c) lo = mid + 1; else hi = mid;
    }
    if (lo < row_ptr[r + 1] && col_idx[lo] == c) {
        *pos = lo;
        return 1;
    }
    return 0;
}

/* csr_to_csrc, csrc_matrix.hpp:44-91. Returns 0 on success; 2 = missing
 * transpose of (err_i, err_j); 3 = row err_i has no diagonal. Arrays sized by
 * the caller (ad n, ia n+1, ja/al/au <= nnz). *value_symmetric set iff every
 * pair matches exactly (au is then left filled but logically elided). */
int oracle_csr_to_csrc(index_t n, const index_t* row_ptr, const index_t* col_idx,
                       const double* values, double* ad, index_t* ia, index_t* ja, double* al,
                       double* au, count_t* k_out, int* value_symmetric, index_t* err_i,
                       index_t* err_j) {
    count_t k = 0;
    int match = 1;
    for (index_t i = 0; i < n; ++i) ad[i] = 0.0;
    ia[0] = 0;
    for (index_t i = 0; i < n; ++i) {
        int has_diag = 0;
        for (index_t q = row_ptr[i]; q < row_ptr[i + 1]; ++q) {
            const index_t j = col_idx[q];
            count_t pos;
            if (j == i) {
                ad[i] = values[q];
                has_diag = 1;
            } else if (j < i) {
                if (!csr_find(row_ptr, col_idx, j, i, &pos)) {
                    *err_i = i;
                    *err_j = j;
                    return 2;
                }
                ja[k] = j;
                al[k] = values[q];
                au[k] = values[pos];
                if (values[pos] != values[q]) match = 0;
                ++k;
            } else {
                if (!csr_find(row_ptr, col_idx, j, i, &pos)) {
                    *err_i = i;
                    *err_j = j;
                    return 2;
                }
            }
        }
        if (!has_diag) {
            *err_i = i;
            *err_j = i;
            return 3;
        }
        ia[i + 1] = (index_t)k;
    }
    *k_out = k;
    *value_symmetric = match;
    return 0;
}

/* ------------------------------------------------------------ scheduling */

static count_t stored_row_count(const index_t* ia, int vs, index_t i) {
    /* partition.hpp:46-49 */
    const count_t pairs = ia[i + 1] - ia[i];
    return 1 + (vs ? pairs : 2 * pairs);
}

/* partition_by_nnz, partition.hpp:55-90 (same double arithmetic). Returns 1
 * when p is out of range [1, n]. */
int oracle_partition_by_nnz(index_t n, const index_t* ia, int vs, int p, index_t* block_start,
                            count_t* block_nnz) {
    if (p < 1 || p > n) return 1;
    count_t* prefix = (count_t*)malloc(sizeof(count_t) * ((size_t)n + 1));
    prefix[0] = 0;
    for (index_t i = 0; i < n; ++i) prefix[i + 1] = prefix[i] + stored_row_count(ia, vs, i);
    const double ideal = (double)prefix[n] / p;
    for (int t = 0; t <= p; ++t) block_start[t] = 0;
    block_start[p] = n;
    index_t b = 0;
    for (int t = 1; t < p; ++t) {
        const double target = t * ideal;
        const index_t lo_bound = block_start[t - 1] + 1;
        const index_t hi_bound = n - (p - t);
        if (b < lo_bound) b = lo_bound;
        while (b < hi_bound && (double)prefix[b] < target) ++b;
        if (b > lo_bound && fabs((double)prefix[b - 1] - target) <= fabs((double)prefix[b] - target))
            --b;
        block_start[t] = b;
    }
    for (int t = 0; t < p; ++t) block_nnz[t] = prefix[block_start[t + 1]] - prefix[block_start[t]];
    free(prefix);
    return 0;
}

/* effective_range(s), partition.hpp:94-109 */
void oracle_effective_ranges(const index_t* ia, const index_t* ja, int p,
                             const index_t* block_start, index_t* lo, index_t* hi) {
    for (int b = 0; b < p; ++b) {
        index_t l = block_start[b];
        for (index_t i = block_start[b]; i < block_start[b + 1]; ++i)
            for (index_t t = ia[i]; t < ia[i + 1]; ++t)
                if (ja[t] < l) l = ja[t];
        lo[b] = l;
        hi[b] = block_start[b + 1] - 1;
    }
}

static int idx_cmp(const void* a, const void* b) {
    index_t x = *(const index_t*)a, y = *(const index_t*)b;
    return x < y ? -1 : (x > y);
}

/* build_interval_plan, partition.hpp:113-134. Outputs: boundaries (<= 2p),
 * intervals (<= 2p) with contributor lists (<= 2p*p). Returns counts. */
void oracle_interval_plan(int p, const index_t* lo, const index_t* hi, index_t* boundaries,
                          int* n_boundaries, index_t* iv_begin, index_t* iv_end,
                          index_t* contrib_ptr, index_t* contrib, int* n_intervals) {
    index_t* cuts = (index_t*)malloc(sizeof(index_t) * (size_t)(2 * p + 1));
    int nc = 0;
    for (int b = 0; b < p; ++b) {
        cuts[nc++] = lo[b];
        cuts[nc++] = hi[b] + 1;
    }
    qsort(cuts, (size_t)nc, sizeof(index_t), idx_cmp);
    int u = 0;
    for (int c = 0; c < nc; ++c)
        if (u == 0 || cuts[u - 1] != cuts[c]) cuts[u++] = cuts[c];
    for (int c = 0; c < u; ++c) boundaries[c] = cuts[c];
    *n_boundaries = u;
    int ni = 0, nct = 0;
    contrib_ptr[0] = 0;
    for (int c = 0; c + 1 < u; ++c) {
        const int before = nct;
        for (int b = 0; b < p; ++b)
            if (lo[b] <= cuts[c] && cuts[c + 1] - 1 <= hi[b]) contrib[nct++] = b;
        if (nct == before) continue;
        iv_begin[ni] = cuts[c];
        iv_end[ni] = cuts[c + 1];
        contrib_ptr[++ni] = nct;
    }
    *n_intervals = ni;
    free(cuts);
}

/* -------------------------------------------------------------- coloring */
/* Literal restatement of coloring.hpp:39-164 for small n: edge sets as a
 * dense n*n byte matrix (direct = 1, indirect = 2), which makes set
 * semantics (no duplicates, direct excluded from indirect) explicit. */

static unsigned char* conflict_matrix(index_t n, const index_t* ia, const index_t* ja, int mode) {
    unsigned char* E = (unsigned char*)calloc((size_t)n * (size_t)n, 1);
    /* direct_conflicts, coloring.hpp:39-45 */
    for (index_t i = 0; i < n; ++i)
        for (index_t t = ia[i]; t < ia[i + 1]; ++t) {
            E[(size_t)ja[t] * n + i] = 1;
            E[(size_t)i * n + ja[t]] = 1;
        }
    if (mode == 0) {
        /* neighborhood, coloring.hpp:55-72: pairs of neighbours of each w */
        for (index_t w = 0; w < n; ++w)
            for (index_t u = 0; u < n; ++u) {
                if (E[(size_t)w * n + u] != 1) continue;
                for (index_t v = u + 1; v < n; ++v) {
                    if (E[(size_t)w * n + v] != 1) continue;
                    if (E[(size_t)u * n + v] == 1) continue;
                    E[(size_t)u * n + v] = 2;
                    E[(size_t)v * n + u] = 2;
                }
            }
    } else {
        /* exact, coloring.hpp:73-89: rows sharing a lower column */
        for (index_t u = 0; u < n; ++u)
            for (index_t v = u + 1; v < n; ++v) {
                if (E[(size_t)u * n + v] == 1) continue;
                int shared = 0;
                for (index_t s = ia[u]; s < ia[u + 1] && !shared; ++s)
                    for (index_t r = ia[v]; r < ia[v + 1]; ++r)
                        if (ja[s] == ja[r]) {
                            shared = 1;
                            break;
                        }
                if (shared) {
                    E[(size_t)u * n + v] = 2;
                    E[(size_t)v * n + u] = 2;
                }
            }
    }
    return E;
}

/* Edge counts of build_conflict_graph (coloring.hpp:93-101). */
void oracle_conflict_edge_counts(index_t n, const index_t* ia, const index_t* ja, int mode,
                                 count_t* n_direct, count_t* n_indirect) {
    unsigned char* E = conflict_matrix(n, ia, ja, mode);
    count_t d = 0, ind = 0;
    for (index_t u = 0; u < n; ++u)
        for (index_t v = u + 1; v < n; ++v) {
            if (E[(size_t)u * n + v] == 1) ++d;
            if (E[(size_t)u * n + v] == 2) ++ind;
        }
    *n_direct = d;
    *n_indirect = ind;
    free(E);
}

/* color_rows, coloring.hpp:119-164: first-fit over direct + indirect edges in
 * natural (0), largest_first (1, stable by degree desc) or smallest_last (2,
 * strict-< lowest-index minimum-degree removal, reversed) order. */
int oracle_color_rows(index_t n, const index_t* ia, const index_t* ja, int mode, int order,
                      int* color) {
    unsigned char* E = conflict_matrix(n, ia, ja, mode);
    count_t* deg = (count_t*)calloc((size_t)n + 1, sizeof(count_t));
    for (index_t u = 0; u < n; ++u)
        for (index_t v = 0; v < n; ++v)
            if (E[(size_t)u * n + v]) ++deg[u];
    index_t* seq = (index_t*)malloc(sizeof(index_t) * ((size_t)n + 1));
    for (index_t i = 0; i < n; ++i) seq[i] = i;
    if (order == 1) {
        /* stable sort by degree descending (insertion sort keeps stability) */
        for (index_t i = 1; i < n; ++i) {
            index_t v = seq[i];
            index_t j = i - 1;
            while (j >= 0 && deg[seq[j]] < deg[v]) {
                seq[j + 1] = seq[j];
                --j;
            }
            seq[j + 1] = v;
        }
    } else if (order == 2) {
        count_t* d = (count_t*)malloc(sizeof(count_t) * ((size_t)n + 1));
        char* removed = (char*)calloc((size_t)n + 1, 1);
        for (index_t i = 0; i < n; ++i) d[i] = deg[i];
        for (index_t step = 0; step < n; ++step) {
            index_t best = -1;
            for (index_t i = 0; i < n; ++i)
                if (!removed[i] && (best < 0 || d[i] < d[best])) best = i;
            removed[best] = 1;
            seq[n - 1 - step] = best; /* reversed removal order */
            for (index_t u = 0; u < n; ++u)
                if (E[(size_t)best * n + u] && !removed[u]) --d[u];
        }
        free(d);
        free(removed);
    }
    for (index_t i = 0; i < n; ++i) color[i] = -1;
    int n_colors = 0;
    char* used = (char*)malloc((size_t)n + 2);
    for (index_t s = 0; s < n; ++s) {
        const index_t v = seq[s];
        memset(used, 0, (size_t)n_colors + 1);
        for (index_t u = 0; u < n; ++u)
            if (E[(size_t)v * n + u] && color[u] >= 0 && color[u] < n_colors + 1) used[color[u]] = 1;
        int c = 0;
        while (used[c]) ++c;
        color[v] = c;
        if (c + 1 > n_colors) n_colors = c + 1;
    }
    free(used);
    free(seq);
    free(deg);
    free(E);
    return n_colors;
}

/* validate_coloring, coloring.hpp:175-198: classes ascending, rows ascending
 * within a class; claim(i) then claim(ja...). Returns 1 if valid, else 0 and
 * the first violation (row_a = previous writer, row_b = current row). */
int oracle_validate_coloring(index_t n, const index_t* ia, const index_t* ja, const int* color,
                             int n_colors, index_t* row_a, index_t* row_b, index_t* position) {
    index_t* writer = (index_t*)malloc(sizeof(index_t) * ((size_t)n + 1));
    for (int c = 0; c < n_colors; ++c) {
        for (index_t q = 0; q < n; ++q) writer[q] = -1;
        for (index_t i = 0; i < n; ++i) {
            if (color[i] != c) continue;
            index_t targets_first = i;
            if (writer[targets_first] >= 0) {
                *row_a = writer[targets_first];
                *row_b = i;
                *position = targets_first;
                free(writer);
                return 0;
            }
            writer[targets_first] = i;
            for (index_t t = ia[i]; t < ia[i + 1]; ++t) {
                const index_t q = ja[t];
                if (writer[q] >= 0) {
                    *row_a = writer[q];
                    *row_b = i;
                    *position = q;
                    free(writer);
                    return 0;
                }
                writer[q] = i;
            }
        }
    }
    free(writer);
    *row_a = *row_b = *position = -1;
    return 1;
}

/* ---------------------------------------------------------------- models */

/* working_set_kb in bytes, working_set.hpp:17-25 */
count_t oracle_working_set_bytes(count_t n, count_t nnz_stored, int value_symmetric) {
    if (value_symmetric) return 12 * nnz_stored + 16 * n + 4;
    return 10 * nnz_stored + 18 * n + 4;
}

/* count_ops, cost_model.hpp:67-89: format 0 csr, 1 csrc, 2 csrc_sym */
void oracle_count_ops(int format, count_t n, count_t nnz_full, count_t* flops, count_t* loads) {
    const count_t k = (nnz_full - n) / 2;
    if (format == 0) {
        *flops = 2 * nnz_full;
        *loads = 3 * nnz_full;
    } else if (format == 1) {
        *flops = 2 * nnz_full - n;
        *loads = 2 * n + 5 * k;
    } else {
        *flops = 2 * nnz_full - n;
        *loads = 2 * n + 4 * k;
    }
}

/* bench_source_vector, bench.hpp:86-90 */
void oracle_bench_source_vector(count_t n, double* x) {
    for (count_t i = 0; i < n; ++i) x[i] = 1.0 + (double)(i % 7) / 7.0;
}

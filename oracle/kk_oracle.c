/*
 * kk_oracle.c -- plain CPU oracle for two-phase SpGEMM C = A*B on CSR matrices.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.  The
 * product path (paper_2103_11991_b200/) never links, imports or calls it, and
 * shares no code, headers or constants with it.
 *
 * What it computes (all citations are lines of /root/reference/PAPER.md):
 *   Eq. (1), PAPER.md:160-163 (Sec. 2.2.1):  C(i,:) = sum_{j in A(i,:)} A(i,j) B(j,:)
 *   symbolic phase:   number of nonzeros per row of C; the
 *                                            last row pointer is nnz(C)
 *   numeric phase,  PAPER.md:168,174:       column indices and values of C
 *   dense accumulator:        "a bit vector for symbolic, and a scalar
 *                                            array for numeric" -- used here for both
 *   compression:              "representing the column indices by bits"
 *   per-row work:         FLOPs per row (multiply-adds)
 *
 * Readings taken where the paper is silent:
 *   R1 structural pattern: an entry exists wherever some A(i,j) and B(j,c) are stored,
 *      whatever its value (explicit and cancelled zeros are kept);
 *   R2 duplicate stored entries are summed, and each stored entry counts as a flop;
 *   R3 rows may be unsorted on input;
 *   R4 output rows are sorted by column;
 *   R5 values accumulate in fp64 in stored order with separate multiply and add
 *      (built with -ffp-contract=off), and bound[c] = sum |a||b| is returned beside.
 *
 * Every loop below follows Gustavson's row-by-row order of Eq. (1); nothing is
 * blocked, fused or reordered.  Row map arrays are int64, column indices int32,
 * values double.  Functions return 0 on success, -1 on an invalid argument
 * (negative sizes, column index out of range, allocation failure).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>
#ifdef _OPENMP
#include <omp.h>
#endif

static int cmp_i32(const void* x, const void* y) {
    int32_t a = *(const int32_t*)x, b = *(const int32_t*)y;
    return (a > b) - (a < b);
}

int kko_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

void kko_set_num_threads(int t) {
#ifdef _OPENMP
    if (t > 0) omp_set_num_threads(t);
#else
    (void)t;
#endif
}

/* flops_i = sum_{p in A(i,:)} nnz(B(A.entries[p], :)).
 * Writes flops[0..m-1]; returns the total, or -1 on a bad column index. */
int64_t kko_row_flops(int64_t m, int64_t n, const int64_t* a_row_map, const int32_t* a_entries,
                      const int64_t* b_row_map, int64_t* flops) {
    int64_t total = 0;
    int bad = 0;
    for (int64_t i = 0; i < m; ++i) {
        int64_t f = 0;
        for (int64_t p = a_row_map[i]; p < a_row_map[i + 1]; ++p) {
            int32_t j = a_entries[p];
            if (j < 0 || j >= n) { bad = 1; continue; }
            f += b_row_map[j + 1] - b_row_map[j];
        }
        flops[i] = f;
        total += f;
    }
    return bad ? -1 : total;
}

/* Compression of B into B_C: each row of B becomes the list of
 * (word = col / 32, mask = OR of 1 << (col % 32)) pairs, one per distinct word,
 * in increasing word order.  bc_row_map (n+1) must be supplied; words/masks must
 * have room for nnz(B) pairs.  This is the canonical form the SPEC examples state
 * (SPEC.md:173-175). */
int kko_compress(int64_t n, int64_t k, const int64_t* b_row_map, const int32_t* b_entries,
                 int64_t* bc_row_map, int32_t* words, uint32_t* masks) {
    int64_t nwords_k = (k + 31) / 32;
    uint32_t* bits = (uint32_t*)calloc((size_t)(nwords_k > 0 ? nwords_k : 1), sizeof(uint32_t));
    if (!bits) return -1;
    int64_t out = 0;
    bc_row_map[0] = 0;
    for (int64_t j = 0; j < n; ++j) {
        for (int64_t q = b_row_map[j]; q < b_row_map[j + 1]; ++q) {
            int32_t c = b_entries[q];
            if (c < 0 || c >= k) { free(bits); return -1; }
            bits[c / 32] |= 1u << (c % 32);
        }
        /* emit the distinct words this row touched, in increasing order */
        int64_t len = b_row_map[j + 1] - b_row_map[j];
        int32_t* wl = (int32_t*)malloc((size_t)(len > 0 ? len : 1) * sizeof(int32_t));
        if (!wl) { free(bits); return -1; }
        for (int64_t q = 0; q < len; ++q) wl[q] = b_entries[b_row_map[j] + q] / 32;
        qsort(wl, (size_t)len, sizeof(int32_t), cmp_i32);
        for (int64_t q = 0; q < len; ++q) {
            if (q > 0 && wl[q] == wl[q - 1]) continue;
            words[out] = wl[q];
            masks[out] = bits[wl[q]];
            bits[wl[q]] = 0;
            ++out;
        }
        free(wl);
        bc_row_map[j + 1] = out;
    }
    free(bits);
    return 0;
}

/* Symbolic phase with the dense bit-vector accumulator
 * (PAPER.md:180): count_i = |union_{j in A(i,:)} cols(B(j,:))|.  Writes
 * c_row_map[0..m] as the exclusive prefix sum of the counts; c_row_map[m] = nnz(C). */
int kko_symbolic(int64_t m, int64_t n, int64_t k, const int64_t* a_row_map, const int32_t* a_entries,
                 const int64_t* b_row_map, const int32_t* b_entries, int64_t* c_row_map) {
    if (m < 0 || n < 0 || k < 0) return -1;
    int64_t* counts = (int64_t*)malloc((size_t)(m > 0 ? m : 1) * sizeof(int64_t));
    if (!counts) return -1;
    int bad = 0;
#pragma omp parallel reduction(| : bad)
    {
        int64_t nwords = (k + 31) / 32;
        uint32_t* bitvec = (uint32_t*)calloc((size_t)(nwords > 0 ? nwords : 1), sizeof(uint32_t));
        if (!bitvec) bad = 1;
#pragma omp for schedule(dynamic, 256)
        for (int64_t i = 0; i < m; ++i) {
            if (!bitvec) continue;
            int64_t cnt = 0;
            for (int64_t p = a_row_map[i]; p < a_row_map[i + 1]; ++p) {
                int32_t j = a_entries[p];
                if (j < 0 || j >= n) { bad = 1; continue; }
                for (int64_t q = b_row_map[j]; q < b_row_map[j + 1]; ++q) {
                    int32_t c = b_entries[q];
                    if (c < 0 || c >= k) { bad = 1; continue; }
                    uint32_t bit = 1u << (c % 32);
                    if (!(bitvec[c / 32] & bit)) {
                        bitvec[c / 32] |= bit;
                        ++cnt;
                    }
                }
            }
            counts[i] = cnt;
            /* reset only the words this row touched */
            for (int64_t p = a_row_map[i]; p < a_row_map[i + 1]; ++p) {
                int32_t j = a_entries[p];
                if (j < 0 || j >= n) continue;
                for (int64_t q = b_row_map[j]; q < b_row_map[j + 1]; ++q) {
                    int32_t c = b_entries[q];
                    if (c >= 0 && c < k) bitvec[c / 32] = 0;
                }
            }
        }
        free(bitvec);
    }
    c_row_map[0] = 0;
    for (int64_t i = 0; i < m; ++i) c_row_map[i + 1] = c_row_map[i] + counts[i];
    free(counts);
    return bad ? -1 : 0;
}

/* Numeric phase (Eq. (1) at PAPER.md:160-163) with the dense
 * scalar-array accumulator.  For each row i, in stored order:
 *     acc[c] = acc[c] + A(i,j) * B(j,c),   bound[c] = bound[c] + |A(i,j)| * |B(j,c)|
 * then the row's distinct columns are sorted (R4) and written at c_row_map[i].
 * c_row_map must be the symbolic result; a row whose distinct-column count
 * differs from c_row_map[i+1]-c_row_map[i] returns -1.  c_bound may be NULL. */
int kko_numeric(int64_t m, int64_t n, int64_t k, const int64_t* a_row_map, const int32_t* a_entries,
                const double* a_values, const int64_t* b_row_map, const int32_t* b_entries,
                const double* b_values, const int64_t* c_row_map, int32_t* c_entries, double* c_values,
                double* c_bound) {
    if (m < 0 || n < 0 || k < 0) return -1;
    int bad = 0;
#pragma omp parallel reduction(| : bad)
    {
        int64_t* marker = (int64_t*)malloc((size_t)(k > 0 ? k : 1) * sizeof(int64_t));
        double* acc = (double*)malloc((size_t)(k > 0 ? k : 1) * sizeof(double));
        double* bnd = (double*)malloc((size_t)(k > 0 ? k : 1) * sizeof(double));
        if (!marker || !acc || !bnd) bad = 1;
        if (marker)
            for (int64_t c = 0; c < k; ++c) marker[c] = -1;
#pragma omp for schedule(dynamic, 256)
        for (int64_t i = 0; i < m; ++i) {
            if (!marker || !acc || !bnd) continue;
            int64_t base = c_row_map[i];
            int64_t len = 0;
            int64_t cap = c_row_map[i + 1] - c_row_map[i];
            for (int64_t p = a_row_map[i]; p < a_row_map[i + 1]; ++p) {
                int32_t j = a_entries[p];
                if (j < 0 || j >= n) { bad = 1; continue; }
                double a = a_values[p];
                for (int64_t q = b_row_map[j]; q < b_row_map[j + 1]; ++q) {
                    int32_t c = b_entries[q];
                    if (c < 0 || c >= k) { bad = 1; continue; }
                    double b = b_values[q];
                    if (marker[c] != i) {
                        marker[c] = i;
                        acc[c] = 0.0;
                        bnd[c] = 0.0;
                        if (len < cap) c_entries[base + len] = c;
                        ++len;
                    }
                    double prod = a * b;
                    acc[c] = acc[c] + prod;
                    bnd[c] = bnd[c] + fabs(a) * fabs(b);
                }
            }
            if (len != cap) { bad = 1; continue; }
            qsort(c_entries + base, (size_t)len, sizeof(int32_t), cmp_i32);
            for (int64_t t = 0; t < len; ++t) {
                int32_t c = c_entries[base + t];
                c_values[base + t] = acc[c];
                if (c_bound) c_bound[base + t] = bnd[c];
            }
        }
        free(marker);
        free(acc);
        free(bnd);
    }
    return bad ? -1 : 0;
}

/*
 * Jacobi-fused SpGEMM reference, PAPER.md:188-217 (Sec. 2.2.2): C = (I - omega D^-1 A) B
 * with A square (m x m), B m x k, dinv[i] = D^-1(i) given.  Written as the paper's
 * three-kernel composition (MSAK), applied row by row (rows are
 * independent):
 *   1. E(i,:) = sum_{j in A(i,:)} A(i,j) B(j,:)          (Eq. 1, usual SpGEMM)
 *   2. F(i,:) = D^-1(i) E(i,:)                             (scaling)
 *   3. C(i,:) = B(i,:) - omega F(i,:)                      (matrix addition)
 * The pattern of C(i,:) is the union of the patterns of B(i,:) and E(i,:) (structural,
 * R1); with a stored diagonal in A it equals E's pattern.  Values:
 * c = b - omega * (dinv_i * e) on the union (b = 0 or e = 0 where a side is absent).
 * bound = |b| + |omega| |dinv_i| sum |a||b| (R5 tolerance reference).
 * kko_jacobi_counts fills counts[m] (|C(i,:)|); kko_jacobi_fill fills the rows given
 * the exclusive scan c_row_map.  Return 0, or -1 on bad input.
 */
static int jacobi_rows(int64_t m, int64_t k, const int64_t* a_row_map, const int32_t* a_entries,
                       const double* a_values, const int64_t* b_row_map, const int32_t* b_entries,
                       const double* b_values, double omega, const double* dinv, int64_t* counts,
                       const int64_t* c_row_map, int32_t* c_entries, double* c_values, double* c_bound) {
    if (m < 0 || k < 0) return -1;
    int bad = 0;
#pragma omp parallel reduction(| : bad)
    {
        int64_t* marker = (int64_t*)malloc((size_t)(k > 0 ? k : 1) * sizeof(int64_t));
        double* e = (double*)malloc((size_t)(k > 0 ? k : 1) * sizeof(double));
        double* eb = (double*)malloc((size_t)(k > 0 ? k : 1) * sizeof(double));
        double* bv = (double*)malloc((size_t)(k > 0 ? k : 1) * sizeof(double));
        int32_t* cols = (int32_t*)malloc((size_t)(k > 0 ? k : 1) * sizeof(int32_t));
        if (!marker || !e || !eb || !bv || !cols) bad = 1;
        if (marker)
            for (int64_t c = 0; c < k; ++c) marker[c] = -1;
#pragma omp for schedule(dynamic, 256)
        for (int64_t i = 0; i < m; ++i) {
            if (!marker || !e || !eb || !bv || !cols) continue;
            int64_t len = 0;
            /* step 1: E(i,:) */
            for (int64_t p = a_row_map[i]; p < a_row_map[i + 1]; ++p) {
                int32_t j = a_entries[p];
                if (j < 0 || j >= m) { bad = 1; continue; }
                double a = a_values ? a_values[p] : 0.0;
                for (int64_t q = b_row_map[j]; q < b_row_map[j + 1]; ++q) {
                    int32_t c = b_entries[q];
                    if (c < 0 || c >= k) { bad = 1; continue; }
                    if (marker[c] != i) {
                        marker[c] = i;
                        e[c] = 0.0;
                        eb[c] = 0.0;
                        bv[c] = 0.0;
                        cols[len++] = c;
                    }
                    if (a_values) {
                        double b = b_values[q];
                        double prod = a * b;
                        e[c] = e[c] + prod;
                        eb[c] = eb[c] + fabs(a) * fabs(b);
                    }
                }
            }
            /* B(i,:) joins the pattern (step 3's addition) */
            for (int64_t q = b_row_map[i]; q < b_row_map[i + 1]; ++q) {
                int32_t c = b_entries[q];
                if (c < 0 || c >= k) { bad = 1; continue; }
                if (marker[c] != i) {
                    marker[c] = i;
                    e[c] = 0.0;
                    eb[c] = 0.0;
                    bv[c] = 0.0;
                    cols[len++] = c;
                }
                if (b_values) bv[c] = bv[c] + b_values[q];
            }
            if (counts) {
                counts[i] = len;
                continue;
            }
            int64_t base = c_row_map[i];
            if (len != c_row_map[i + 1] - base) { bad = 1; continue; }
            qsort(cols, (size_t)len, sizeof(int32_t), cmp_i32);
            for (int64_t t = 0; t < len; ++t) {
                int32_t c = cols[t];
                double f = dinv[i] * e[c];          /* step 2 */
                c_entries[base + t] = c;
                c_values[base + t] = bv[c] - omega * f; /* step 3 */
                if (c_bound) c_bound[base + t] = fabs(bv[c]) + fabs(omega) * fabs(dinv[i]) * eb[c];
            }
        }
        free(marker);
        free(e);
        free(eb);
        free(bv);
        free(cols);
    }
    return bad ? -1 : 0;
}

int kko_jacobi_counts(int64_t m, int64_t k, const int64_t* a_row_map, const int32_t* a_entries,
                      const int64_t* b_row_map, const int32_t* b_entries, int64_t* counts) {
    return jacobi_rows(m, k, a_row_map, a_entries, NULL, b_row_map, b_entries, NULL, 0.0, NULL, counts, NULL,
                       NULL, NULL, NULL);
}

int kko_jacobi_fill(int64_t m, int64_t k, const int64_t* a_row_map, const int32_t* a_entries,
                    const double* a_values, const int64_t* b_row_map, const int32_t* b_entries,
                    const double* b_values, double omega, const double* dinv, const int64_t* c_row_map,
                    int32_t* c_entries, double* c_values, double* c_bound) {
    return jacobi_rows(m, k, a_row_map, a_entries, a_values, b_row_map, b_entries, b_values, omega, dinv, NULL,
                       c_row_map, c_entries, c_values, c_bound);
}

/*
 * SpAdd reference, PAPER.md:263-267 (Sec. 2.3): C = alpha A + beta B on CSR matrices of
 * the same shape, with entries of equal (row, column) merged -- also duplicates inside
 * A or B ("if row i of A contains many entries for column j, these entries will be
 * additively merged into a single entry C(i,j)").  Inputs may be unsorted.
 * Written as the plain definition with the dense accumulator (one marker per column):
 * for each row, every stored entry of A then of B adds alpha*a (beta*b) to its column.
 * Output rows sorted (R4); structural pattern (R1: cancellations kept); bound =
 * |alpha| sum|a| + |beta| sum|b| per entry.
 * kko_spadd_counts: counts[m]; kko_spadd_fill: entries/values/bound given c_row_map.
 */
static int spadd_rows(int64_t m, int64_t k, const int64_t* a_row_map, const int32_t* a_entries,
                      const double* a_values, const int64_t* b_row_map, const int32_t* b_entries,
                      const double* b_values, double alpha, double beta, int64_t* counts,
                      const int64_t* c_row_map, int32_t* c_entries, double* c_values, double* c_bound) {
    if (m < 0 || k < 0) return -1;
    int bad = 0;
#pragma omp parallel reduction(| : bad)
    {
        int64_t* marker = (int64_t*)malloc((size_t)(k > 0 ? k : 1) * sizeof(int64_t));
        double* acc = (double*)malloc((size_t)(k > 0 ? k : 1) * sizeof(double));
        double* bnd = (double*)malloc((size_t)(k > 0 ? k : 1) * sizeof(double));
        int32_t* cols = (int32_t*)malloc((size_t)(k > 0 ? k : 1) * sizeof(int32_t));
        if (!marker || !acc || !bnd || !cols) bad = 1;
        if (marker)
            for (int64_t c = 0; c < k; ++c) marker[c] = -1;
#pragma omp for schedule(dynamic, 256)
        for (int64_t i = 0; i < m; ++i) {
            if (!marker || !acc || !bnd || !cols) continue;
            int64_t len = 0;
            for (int side = 0; side < 2; ++side) {
                const int64_t* rm = side ? b_row_map : a_row_map;
                const int32_t* en = side ? b_entries : a_entries;
                const double* va = side ? b_values : a_values;
                const double s = side ? beta : alpha;
                for (int64_t p = rm[i]; p < rm[i + 1]; ++p) {
                    int32_t c = en[p];
                    if (c < 0 || c >= k) { bad = 1; continue; }
                    if (marker[c] != i) {
                        marker[c] = i;
                        acc[c] = 0.0;
                        bnd[c] = 0.0;
                        cols[len++] = c;
                    }
                    if (va) {
                        double prod = s * va[p];
                        acc[c] = acc[c] + prod;
                        bnd[c] = bnd[c] + fabs(s) * fabs(va[p]);
                    }
                }
            }
            if (counts) {
                counts[i] = len;
                continue;
            }
            int64_t base = c_row_map[i];
            if (len != c_row_map[i + 1] - base) { bad = 1; continue; }
            qsort(cols, (size_t)len, sizeof(int32_t), cmp_i32);
            for (int64_t t = 0; t < len; ++t) {
                c_entries[base + t] = cols[t];
                c_values[base + t] = acc[cols[t]];
                if (c_bound) c_bound[base + t] = bnd[cols[t]];
            }
        }
        free(marker);
        free(acc);
        free(bnd);
        free(cols);
    }
    return bad ? -1 : 0;
}

int kko_spadd_counts(int64_t m, int64_t k, const int64_t* a_row_map, const int32_t* a_entries,
                     const int64_t* b_row_map, const int32_t* b_entries, int64_t* counts) {
    return spadd_rows(m, k, a_row_map, a_entries, NULL, b_row_map, b_entries, NULL, 0.0, 0.0, counts, NULL, NULL,
                      NULL, NULL);
}

int kko_spadd_fill(int64_t m, int64_t k, const int64_t* a_row_map, const int32_t* a_entries,
                   const double* a_values, const int64_t* b_row_map, const int32_t* b_entries,
                   const double* b_values, double alpha, double beta, const int64_t* c_row_map,
                   int32_t* c_entries, double* c_values, double* c_bound) {
    return spadd_rows(m, k, a_row_map, a_entries, a_values, b_row_map, b_entries, b_values, alpha, beta, NULL,
                      c_row_map, c_entries, c_values, c_bound);
}

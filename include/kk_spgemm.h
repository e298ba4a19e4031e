/*
 * kk_spgemm.h -- C ABI of the B200 two-phase hash SpGEMM, C = A * B on CSR matrices.
 *
 * The calls follow the paper's statement of the two-phase protocol
 * (Sec. 2.2.1):
 *   "we first allocate the row pointers of C"            -> caller allocates c_row_map
 *   "We may compress B into B_C"                          -> inside kk_spgemm_symbolic
 *   "perform the symbolic phase on A and B_C to fill the row pointers array"
 *                                                         -> kk_spgemm_symbolic
 *   "The last entry of the row pointers array amounts to ... nnz(C)"
 *                                                         -> *c_nnz (host) on return
 *   "Then we allocate two more arrays ... of size nnz(C)" -> caller allocates entries/values
 *   "Finally, we perform the numeric phase"               -> kk_spgemm_numeric
 * and the kernel handle of PAPER.md:708-712 (Sec. 6: variant choice and symbolic
 * state carried between the phases).
 *
 * Conventions (all functions):
 *   - Matrix arrays (row_map, entries, values) are DEVICE pointers on the handle's
 *     device.  The library never takes ownership of them.
 *   - row_map has nrows+1 entries of `offset_type` (int32 or int64); A, B and C use
 *     the same offset type.  entries are int32 column indices.  values are float
 *     or double, the same type for A, B and C.  Rows may be unsorted and may hold
 *     duplicate columns (duplicates are summed).
 *   - C's pattern is the structural product: an entry exists wherever a stored
 *     A(i,j) meets a stored B(j,c), whatever the value (cancelled zeros are kept).
 *   - All device work is enqueued on `stream` (a cudaStream_t, 0 = legacy default).
 *     kk_spgemm_symbolic synchronises `stream` twice: once to read the row-bin sizes
 *     (so empty bins are not launched and grids fit their bins) and once to return
 *     nnz(C) to the host.
 *     kk_spgemm_numeric is fully asynchronous.
 *   - Errors are returned as kk_status_t; nothing is thrown across the ABI.  On an
 *     error, kk_last_error_detail() gives a one-line description.
 *   - A handle is not thread-safe; distinct handles are independent.
 */
#ifndef KK_SPGEMM_H
#define KK_SPGEMM_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    KK_OK = 0,
    KK_ERR_INVALID_ARG = 1,      /* null pointer, negative size, bad option value */
    KK_ERR_DIM_MISMATCH = 2,     /* A.ncols != B.nrows */
    KK_ERR_UNSUPPORTED_TYPE = 3, /* mixed offset or value types */
    KK_ERR_INDEX_OVERFLOW = 4,   /* nnz(C) > INT32_MAX with int32 offsets; or column index
                                    out of range when opts.validate = 1 */
    KK_ERR_STALE_HANDLE = 5,     /* numeric called without a matching symbolic */
    KK_ERR_OUT_OF_MEMORY = 6,    /* workspace allocation failed */
    KK_ERR_CUDA = 7              /* CUDA launch or runtime error */
} kk_status_t;

typedef enum { KK_I32 = 0, KK_I64 = 1 } kk_index_t;
typedef enum { KK_F32 = 0, KK_F64 = 1 } kk_scalar_t;

/* A CSR matrix ("CrsMatrix" / "StaticCrsGraph"); device pointers. */
typedef struct {
    int64_t nrows;
    int64_t ncols;
    int64_t nnz;              /* = row_map[nrows] */
    kk_index_t offset_type;   /* type of row_map */
    kk_scalar_t value_type;   /* type of values */
    const void* row_map;      /* nrows+1 offsets */
    const int32_t* entries;   /* nnz column indices */
    const void* values;       /* nnz values (may be NULL for symbolic-only use) */
} kk_csr_t;

typedef struct kk_spgemm_handle_s* kk_spgemm_handle_t;

/* Workspace allocator: alloc(bytes, stream, ctx) returns device memory usable on
 * `stream`; free(ptr, bytes, stream, ctx) releases it.  NULL = cudaMallocAsync /
 * cudaFreeAsync.  The handle grows its workspace monotonically and frees it in
 * kk_spgemm_destroy. */
typedef void* (*kk_alloc_fn)(size_t bytes, void* stream, void* ctx);
typedef void (*kk_free_fn)(void* ptr, size_t bytes, void* stream, void* ctx);

typedef struct {
    int sort_rows;     /* 1 (default): C rows sorted by column; 0: any order within a row */
    int compression;   /* -1 (default) auto, 0 off, 1 on: compress B into B_C */
    int validate;      /* 1: check column indices of A and B are in range (error otherwise) */
    int num_streams;   /* internal streams used to overlap work bins (default 2, 1 = none) */
    int timing;        /* 1: bracket every kernel launch with CUDA events on the stream it is
                          launched on (read with kk_spgemm_kernel_times); default 0 */
    int patterns;      /* 1 (default): symbolic keeps the compressed pattern of rows that fit
                          (sorted (word, mask) pairs, <= 64 words) in the handle, and numeric
                          accumulates those rows by rank lookup; 0: numeric re-derives every
                          row.  Costs up to 48 * 8 bytes of workspace per row of A. */
    int deterministic; /* 1: bitwise-reproducible values from run to run (the handle-selected
                          variant of PAPER.md:708-712): the tiers that would add products into
                          a shared or global accumulator with atomics (long rows, short-B-row
                          warp tables) add them in A-entry order instead.  Needs strictly
                          increasing B rows (then every other tier is order-fixed already);
                          otherwise kk_spgemm_symbolic returns KK_ERR_UNSUPPORTED_TYPE.
                          Default 0 (long rows are slower in this mode). */
    kk_alloc_fn alloc;
    kk_free_fn free;
    void* alloc_ctx;
} kk_spgemm_opts_t;

#define KK_STATS_MAX_BINS 24

typedef struct {
    int64_t muladds;          /* sum_i sum_{j in A(i,:)} nnz(B(j,:)) */
    int64_t nnz_c;            /* row_map[m] of the last symbolic */
    int64_t compressed_words; /* |B_C| (0 when compression was not used) */
    int compression_used;     /* 1 if the last symbolic ran on B_C */
    int b_sorted;             /* 1 if every row of B was non-decreasing */
    int b_strict;             /* 1 if every row of B was strictly increasing */
    int num_symbolic_bins;
    int num_numeric_bins;
    int64_t symbolic_bin_rows[KK_STATS_MAX_BINS]; /* rows per symbolic work bin (num_symbolic_bins used) */
    int64_t numeric_bin_rows[KK_STATS_MAX_BINS];  /* rows per numeric work bin (num_numeric_bins used) */
    int64_t kernel_launches;  /* total kernels this handle launched since creation */
    int64_t workspace_bytes;  /* bytes currently held */
} kk_spgemm_stats_t;

/* Fill *opts with the defaults listed above. */
void kk_spgemm_opts_default(kk_spgemm_opts_t* opts);

/* Create a handle on CUDA device `device` (>= 0).  opts may be NULL (defaults). */
kk_status_t kk_spgemm_create(kk_spgemm_handle_t* handle, int device, const kk_spgemm_opts_t* opts);

/* Release the handle and its workspace (after synchronising its device work). */
kk_status_t kk_spgemm_destroy(kk_spgemm_handle_t handle);

/* Step a1+a2 (per-row FLOPs, parallel prefix sum):
 * flops[i] = sum_{j in A(i,:)} nnz(B(j,:)) (device, m int64, may be NULL);
 * flops_scan = exclusive prefix of flops (device, m+1 int64, may be NULL);
 * *total (host, may be NULL) = flops_scan[m] -- synchronises `stream` when non-NULL.
 * Used for flop-balanced row partitioning across GPUs. */
kk_status_t kk_spgemm_row_flops(kk_spgemm_handle_t handle, const kk_csr_t* A, const kk_csr_t* B,
                                int64_t* flops, int64_t* flops_scan, int64_t* total, void* stream);

/* Step a4 ("compress B into B_C by representing the column indices by
 * bits"): for each row j of B, writes len[j] (device, n int32) pairs
 * (word = col >> 5, mask = OR of 1 << (col & 31)) at pairs[B.row_map[j] ...]
 * (device, capacity nnz(B) uint64, word in the low 32 bits, mask in the high 32).
 * Adjacent equal words are merged; on sorted rows this is the canonical form
 * (distinct increasing words).  Exposed for tests; symbolic calls it internally. */
kk_status_t kk_spgemm_compress(kk_spgemm_handle_t handle, const kk_csr_t* B, int32_t* len, uint64_t* pairs,
                               void* stream);

/* Symbolic phase: fills c_row_map (device, A.nrows+1 entries of
 * A.offset_type, caller-allocated) with the row pointers of C and returns nnz(C) in
 * *c_nnz (host).  Runs flop count, scan, binning, compression and the per-bin
 * symbolic kernels; the handle keeps the row bins for the numeric phase. */
kk_status_t kk_spgemm_symbolic(kk_spgemm_handle_t handle, const kk_csr_t* A, const kk_csr_t* B,
                               void* c_row_map, int64_t* c_nnz, void* stream);

/* Numeric phase (Eq. (1) at PAPER.md:160-163): writes the column
 * indices (c_entries, device, nnz(C) int32) and values (c_values, device, nnz(C) of
 * A.value_type) of C.  c_row_map must be the array filled by the last symbolic call
 * on the same A/B patterns (same sizes, pointers and types), else
 * KK_ERR_STALE_HANDLE.  The values of A and B may change between calls
 * (symbolic reuse). */
kk_status_t kk_spgemm_numeric(kk_spgemm_handle_t handle, const kk_csr_t* A, const kk_csr_t* B,
                              const void* c_row_map, int32_t* c_entries, void* c_values, void* stream);

/* Jacobi-fused numeric phase (Sec. 2.2.2; Eq. (2) at PAPER.md:209-211):
 * C = (I - omega D^-1 A) B, i.e. C(i,:) = B(i,:) - omega * dinv[i] * E(i,:) with
 * E(i,:) = sum_{j in A(i,:)} A(i,j) B(j,:).  Runs after kk_spgemm_symbolic(A, B) -- the
 * usual symbolic, as in the paper (pattern(C) = pattern(E) because A(i,i) is stored) --
 * and writes c_entries / c_values exactly like kk_spgemm_numeric.
 *   omega: the scalar (host); dinv: device, A.nrows values of A.value_type, the entries
 *   of D^-1 (caller-owned, read only).
 * Preconditions: A square (A.nrows == A.ncols == B.nrows, else KK_ERR_DIM_MISMATCH);
 * every row of A stores its diagonal entry -- checked only when
 * opts.validate = 1 (KK_ERR_INVALID_ARG); without it, entries of B(i,:) outside E(i,:)'s
 * pattern are dropped.  Every tier has the fused form, the long-row (dense) tiers included:
 * per row the kernel forms -omega * dinv[i] once, scales E(i,:) by it and inserts B(i,:)
 * into the accumulator (the paper's fusion).
 * Asynchronous on `stream` (the validate check synchronises it). */
kk_status_t kk_spgemm_jacobi_numeric(kk_spgemm_handle_t handle, double omega, const void* dinv, const kk_csr_t* A,
                                     const kk_csr_t* B, const void* c_row_map, int32_t* c_entries, void* c_values,
                                     void* stream);

/* SpAdd symbolic (Sec. 2.3.1, Alg. 1): C = alpha A + beta B for A, B of
 * the same shape (else KK_ERR_DIM_MISMATCH) and offset type.  Fills c_row_map (device,
 * A.nrows+1 of A.offset_type, caller-allocated), returns nnz(C) in *c_nnz (host), and keeps
 * in the handle the scatter position of every entry of A and B in its row of C (the
 * paper's Apos / Bpos).  Rows may be unsorted and unmerged (duplicate columns inside A or
 * B are merged into one entry of C); C's pattern is the structural union.  A warp owns a row
 * of nnz(A_i) + nnz(B_i) <= 256 (register bitonic sort / merge), a CTA a longer row (shared-
 * memory bitonic sort); rows with nnz(A_i) + nnz(B_i) > 16384 return
 * KK_ERR_UNSUPPORTED_TYPE.  Synchronises `stream`. */
kk_status_t kk_spadd_symbolic(kk_spgemm_handle_t handle, const kk_csr_t* A, const kk_csr_t* B, void* c_row_map,
                              int64_t* c_nnz, void* stream);

/* SpAdd numeric: writes C's sorted column indices (c_entries, device, nnz(C)
 * int32) and values alpha*a + beta*b (c_values, device, A.value_type) by scattering A's and
 * B's entries to the positions kept by kk_spadd_symbolic on the same patterns (same sizes,
 * pointers, types, row map; else KK_ERR_STALE_HANDLE).  Values may change between calls.
 * Asynchronous on `stream`. */
kk_status_t kk_spadd_numeric(kk_spgemm_handle_t handle, double alpha, const kk_csr_t* A, double beta,
                             const kk_csr_t* B, const void* c_row_map, int32_t* c_entries, void* c_values,
                             void* stream);

/* Fused Galerkin triple product Ac = R * A * P (multigrid coarse operator, the SpGEMM use the
 * paper motivates at PAPER.md:152, 200), in one pass without forming A*P:
 * Ac(I,c) = sum_{i in R(I,:)} R(I,i) sum_{j in A(i,:)} A(i,j) P(j,c).  R: mc x m, A: m x n,
 * P: n x nc (else KK_ERR_DIM_MISMATCH), device CSR of one offset type and one value type.
 * kk_spgemm_rap_symbolic fills c_row_map (device, mc+1 of R.offset_type, caller-allocated)
 * and returns nnz(Ac) in *c_nnz (host; synchronises `stream`); rows of Ac with more than 256
 * distinct columns return KK_ERR_UNSUPPORTED_TYPE (compute them as two products).
 * kk_spgemm_rap_numeric writes Ac's sorted column indices and values (device, caller-
 * allocated, nnz(Ac)) for the matrices and row map of the last rap symbolic on this handle
 * (else KK_ERR_STALE_HANDLE); values of R, A, P may change between calls.  Asynchronous. */
kk_status_t kk_spgemm_rap_symbolic(kk_spgemm_handle_t handle, const kk_csr_t* R, const kk_csr_t* A,
                                   const kk_csr_t* P, void* c_row_map, int64_t* c_nnz, void* stream);
kk_status_t kk_spgemm_rap_numeric(kk_spgemm_handle_t handle, const kk_csr_t* R, const kk_csr_t* A,
                                  const kk_csr_t* P, const void* c_row_map, int32_t* c_entries, void* c_values,
                                  void* stream);

/* C = A*B with A, B and C in HOST memory: the paper's protocol run end to
 * end over host buffers.  A, B: CSR whose row_map / entries / values are HOST pointers
 * (pinned memory, e.g. cudaHostAlloc, lets the copies run asynchronously; pageable memory
 * works but serialises them).  A is processed in contiguous row blocks (row blocks are
 * independent products, Eq. 1 at PAPER.md:160-163): each block's host->device copies, symbolic
 * + numeric phases and device->host copy of its rows of C overlap the neighbouring blocks' on
 * four streams.  `blocks` > 0 fixes the block count (with 4 or more the first two are a quarter
 * and a half of the others); `blocks` <= 0 with A of >= 65,536 rows runs a small first block
 * (1/64 of the rows) and plans the rest from its output size, about 48 MB of host<->device
 * traffic per block (env KK_HOST_BLOCK_BYTES overrides); fewer rows: one block.  B is copied
 * once, in 16 row chunks; a block whose columns all lie in a prefix of B's rows starts as soon
 * as that prefix has arrived.  When A and B are the same host matrix (same three pointers), A's
 * rows are taken from B's device copy instead of crossing PCIe twice.  Outputs:
 *   c_row_map: HOST, A.nrows+1 of A.offset_type, caller-allocated, filled with C's row map;
 *   *c_nnz: nnz(C);
 *   *c_entries, *c_values: HOST (pinned) arrays of nnz(C) column indices / values owned by the
 *     handle, valid until the next kk_spgemm_multiply_host or kk_spgemm_destroy.
 * Errors as kk_spgemm_symbolic / numeric; KK_ERR_INDEX_OVERFLOW when nnz(C) does not fit
 * int32 offsets.  Synchronises `stream` (returns when C is on the host). */
kk_status_t kk_spgemm_multiply_host(kk_spgemm_handle_t handle, const kk_csr_t* A, const kk_csr_t* B,
                                    void* c_row_map, int64_t* c_nnz, int32_t** c_entries, void** c_values,
                                    int blocks, void* stream);

/* Per-kernel device times (opts.timing = 1).  One record per kernel (or fixed group of
 * launches, e.g. the three launches of a scan), accumulated since the last
 * kk_spgemm_timing_reset: number of launches, total and maximum duration in ms, from
 * CUDA events recorded on the launching stream.  Synchronises on those events.
 * Writes min(*count_inout, number of records) records into `out` (host) and sets
 * *count_inout to the number of records available. */
typedef struct {
    char name[48];
    int64_t launches;
    double total_ms;
    double max_ms;
} kk_kernel_time_t;
kk_status_t kk_spgemm_kernel_times(kk_spgemm_handle_t handle, kk_kernel_time_t* out, int* count_inout);
/* Drop the accumulated kernel times (after synchronising the pending events). */
kk_status_t kk_spgemm_timing_reset(kk_spgemm_handle_t handle);

/* Statistics of the last symbolic/numeric pair. */
kk_status_t kk_spgemm_stats(kk_spgemm_handle_t handle, kk_spgemm_stats_t* stats);

const char* kk_status_string(kk_status_t status);
const char* kk_last_error_detail(kk_spgemm_handle_t handle);

#ifdef __cplusplus
}
#endif

#endif /* KK_SPGEMM_H */

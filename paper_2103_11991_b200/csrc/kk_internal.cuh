// kk_internal.cuh -- internal declarations shared by kk_kernels.cu and kk_api.cu.
//
// Product code only: nothing here is shared with oracle/ (DESIGN.md "Boundary").
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace kk {

constexpr int NB = 18;                       // max work bins per phase
constexpr uint32_t EMPTY = 0xffffffffu;      // empty hash slot (column indices are < 2^31)

// Symbolic bins (by an upper bound ub_i of distinct keys of row i):
//   0: ub = 0 (empty row, no kernel); b = 1..7: warp-owned shared hash with S = 32 << b
//   slots (ub <= S); 8: CTA-owned dense bit-vector window.
constexpr int SYM_WARP_BINS = 7;
constexpr int SYM_DENSE_BIN = 8;
// 9..15: warp-owned dense bit vector over the row's column window [wlo, wlo + W) with
// W = 8K, 16K, 32K, 48K, 64K, 128K, 192K bits (sorted B only; the window comes from the
// first/last column of each B row, "bit vector for symbolic")
constexpr int SYM_WIN_BIN0 = 9;
constexpr int SYM_WIN_NBINS = 7;
// 16: tiny rows (flops_i <= TINY_MAX): a lane owns a row, its columns in registers
constexpr int SYM_TINY_BIN = 16;
constexpr int SYM_NBINS = 17;
constexpr int TINY_MAX = 16;
// Numeric bins (by exact nnz(C_i)):
//   0: empty; b = 1..5: warp-owned shared hash with S = 32 << b slots (nnz <= S/2);
//   6: CTA-owned dense scalar window (column-windowed dense accumulator).
constexpr int NUM_WARP_BINS = 5;
constexpr int NUM_DENSE_BIN = 6;
//   7..11: rows with a pattern kept by symbolic (nnz <= 32 << (b - 7)): word-table rank
//   lookup into a dense per-row value array (no claims, no sort)
//   12..15: the same for patterns whose words span > 2048 words (hashed word lookup;
//   nnz <= 64 << (b - 12))
constexpr int NUM_PAT_BIN0 = 7;
constexpr int NUM_PATH_BIN0 = 12;
constexpr int PAT_DENSE_WORDS = 2048;  // widest word span of a pattern with a dense word index
//   16: tiny rows (flops_i <= TINY_MAX), lane-owned register lists
constexpr int NUM_TINY_BIN = 16;
constexpr int NUM_NBINS = 17;

// Device-side status block.  Written by the kernels, copied to pinned host memory at the
// end of the symbolic phase (the phase's second device->host sync; the first reads the
// symbolic bin sizes after binning).
struct DevStatus {
    unsigned long long total_flops;   // sum_i flops_i
    unsigned long long total_words;   // |B_C| (pairs written by compression)
    unsigned long long nnz_c;         // row_map[m]
    unsigned long long pat_used;      // pairs taken from the row-pattern pool
    int b_sorted;                     // every B row non-decreasing
    int b_strict;                     // every B row strictly increasing
    int bad_index;                    // validate: a column index out of range
    int overflow;                     // int32 row map cannot hold nnz(C)
    int use_comp;                     // symbolic ran on B_C
    int pad;
    int sym_bin_start[NB + 1];        // row ranges of the symbolic bins in perm_sym
    int num_bin_start[NB + 1];        // row ranges of the numeric bins in perm_num
};

// Row patterns kept by the symbolic window kernels for the numeric phase: the sorted
// (word, mask) pairs of row i are pat[off[i] .. off[i] + len[i]); off[i] = -1: none.
struct PatOut {
    uint2* pat;
    long long cap;
    long long* off;
    int* len;
};

struct MatView {
    int64_t nrows, ncols, nnz;
    const void* row_map;
    const int32_t* entries;
    const void* values;
};

// Optional per-kernel CUDA-event timing (kk_spgemm_opts_t.timing; kk_api.cu).
struct KTimer;
void ktimer_begin(KTimer* t, const char* name, cudaStream_t s);
void ktimer_end(KTimer* t, cudaStream_t s);

struct Launch {
    cudaStream_t stream;
    int num_sms;
    long long* launches;   // incremented once per kernel launch
    KTimer* timer;         // null unless timing is on
    // bracket every launch (or fixed group of launches) with begin/end
    void begin(const char* name, cudaStream_t s) const {
        if (timer) ktimer_begin(timer, name, s);
    }
    void end(cudaStream_t s, int nlaunch = 1) const {
        *launches += nlaunch;
        if (timer) ktimer_end(timer, s);
    }
};

// ---- host launchers (kk_kernels.cu) -------------------------------------------------
// B-row flags already established for a prefix of B's rows (the host-buffer product compresses
// only the rows each block adds); default: none
struct StatusCarry {
    int b_sorted = 1, b_strict = 1, bad_index = 0;
    unsigned long long total_words = 0;
};
void init_status(Launch& L, DevStatus* st, const StatusCarry* carry = nullptr);
// bmeta (may be null): per B row {nnz, |B_C row|, first column, last column}
// (first/last = INT_MAX / -1 for empty rows).  Rows [row0, B.nrows) only (the outputs of the
// rows before are kept).
void check_compress(Launch& L, bool off64, const MatView& B, int64_t k, bool do_comp, bool validate,
                    int32_t* bc_len, uint2* pairs, int4* bmeta, DevStatus* st, int64_t row0 = 0);
// bmeta (may be null: then the B row map is read); wlo (may be null): word-aligned first
// column of the window of rows in window bins
void row_flops_bin(Launch& L, bool off64, const MatView& A, const MatView& B, int64_t k, int comp_mode,
                   bool validate, const int32_t* bc_len, const int4* bmeta, int64_t* flops, uint8_t* binid,
                   int32_t* counts, int32_t* wlo, DevStatus* st, long long* pat_off = nullptr);
// exclusive scan of in[0..m) (int32 or int64) into out[0..m] (int32 or int64);
// *total_dst (device, may be null) receives the sum; *overflow set when out is
// int32 and the sum exceeds INT32_MAX.  partial: >= scan_partial_len(m) int64.
int64_t scan_partial_len(int64_t m);
// out != null: out[0..n) = p[...] + delta instead (out may be mapped pinned host memory)
void add_offset(Launch& L, bool off64, void* p, int64_t n, int64_t delta, void* out = nullptr);
// one launch: rm_dst[0..nrm) = rm_src[...] - base, e_dst/v_dst = e_src/v_src (bytes)
void copy_rows(Launch& L, bool off64, void* rm_dst, const void* rm_src, int64_t nrm, int64_t base, void* e_dst,
               const void* e_src, int64_t e_bytes, void* v_dst, const void* v_src, int64_t v_bytes);
// dst[i] = src[i] - base for i < n (offsets of the row map's type; dst may be src)
void rebase_row_map(Launch& L, bool off64, void* dst, const void* src, int64_t n, int64_t base);
void exclusive_scan(Launch& L, bool in64, const void* in, bool out64, void* out, int64_t m, int64_t* partial,
                    unsigned long long* total_dst, int* overflow);
// pat_off (may be null): rows with a stored pattern (and strictly sorted B) go to the
// pattern bins NUM_PAT_BIN0 + (b - 1)
// flops (may be null): rows with flops_i <= TINY_MAX go to NUM_TINY_BIN
void numeric_binid(Launch& L, int64_t m, const int32_t* counts, const long long* pat_off, const int* pat_len,
                   const uint2* pat, const int64_t* flops, uint8_t* binid, const DevStatus* st);
// stable binning of rows by binid: perm lists rows of bin 0, then bin 1, ...
// (each bin in increasing row order); bin_start_dst (device int[NB+1]).
int64_t bin_scratch_len(int64_t m);
void bin_rows(Launch& L, int64_t m, const uint8_t* binid, int32_t* scratch, int32_t* perm, int* bin_start_dst);

struct SymArgs {
    bool off64;
    MatView A, B;
    int64_t k;
    const int32_t* bc_len;
    const uint2* pairs;
    const int32_t* perm;
    const int* bin_start;   // device
    const int* host_bin_start;  // host copy, or null (then every bin is launched)
    const int32_t* wlo;     // window start per row (window bins)
    PatOut pat;             // row-pattern pool (pat.pat may be null: keep none)
    int32_t* counts;
    int32_t* cursors;       // nnz(A) scratch for windowed rows
    const DevStatus* st;
    int logG;
    int comp_mode;          // opts.compression: 1 on, 0 off, -1 decided on the device (a1)
    int* retry = nullptr;   // device int[m + 8]: per-bin lists of rows the speculative small tables gave up on
};
void symbolic_bins(Launch& L, const SymArgs& a, cudaStream_t dense_stream);

struct NumArgs {
    bool off64, f64, sort;
    bool strict;                 // every B row strictly increasing (host copy of the a4 flag)
    bool sorted;                 // every B row non-decreasing (host copy of the a4 flag)
    bool det = false;            // opts.deterministic: products added in A-entry order
    // 1-D linear texture objects over B.entries / B.values (0: none; the pattern tier then
    // loads B with LDG)
    unsigned long long tex_ent = 0, tex_val = 0;
    int* work_ctr = nullptr;     // device scratch: dynamic row counters of the cluster tier
    MatView A, B;
    int64_t k;
    const void* c_row_map;
    int32_t* c_entries;
    void* c_values;
    const int32_t* perm;
    const int* bin_start;        // device
    const int* host_bin_start;   // host copy (row counts known after symbolic)
    int32_t* cursors;
    const DevStatus* st;
    int logG;
    const int32_t* wlo;          // window start per row (pattern rows)
    const uint2* pat;            // row patterns (see PatOut)
    const long long* pat_off;
    const int* pat_len;
    // Jacobi-fused numeric: C = (I - omega D^-1 A) B when dinv != null
    const void* dinv = nullptr;  // device, A.nrows values of the value type
    double omega = 0.0;
};
void numeric_bins(Launch& L, const NumArgs& a, cudaStream_t dense_stream);
// SpAdd (kk_spadd.cu): symbolic fills counts[m], apos[nnzA], bpos[nnzB], dup[m] (row has
// an unmerged column); *too_long (device) set when a row has nnz(A_i) + nnz(B_i) > 256
void spadd_symbolic(Launch& L, bool off64, int64_t m, const MatView& A, const MatView& B, int32_t* counts,
                    int32_t* apos, int32_t* bpos, uint8_t* dup, int* too_long);
void spadd_numeric(Launch& L, bool off64, bool f64, int64_t m, double alpha, const MatView& A, double beta,
                   const MatView& B, const void* crm, int32_t* cent, void* cval, const int32_t* apos,
                   const int32_t* bpos, const uint8_t* dup);
// Fused triple product Ac = R*A*P (kk_rap.cu): symbolic fills counts[R.nrows] and sets
// *too_many (device) when a coarse row has more distinct columns than the warp table holds
void rap_symbolic(Launch& L, bool off64, const MatView& R, const MatView& A, const MatView& P, int32_t* counts,
                  int* too_many);
void rap_numeric(Launch& L, bool off64, bool f64, const MatView& R, const MatView& A, const MatView& P,
                 const void* crm, int32_t* cent, void* cval);
// validate for the Jacobi-fused numeric: *missing (mapped pinned host int, missing_map its
// device address) = rows of the square A without a stored diagonal entry; scratch: one device
// int.  Synchronises L.stream.  false on a CUDA error.
bool check_diagonal(Launch& L, bool off64, int64_t m, const void* row_map, const int32_t* entries, int* scratch,
                    int* missing, int* missing_map);
// dst[g][0 .. bytes[g]/4) = src[g][...] for g < nseg <= 4, by one CTA's stores (dst may be the
// device address of mapped pinned host memory: a status read without a copy engine)
void post_words(Launch& L, int nseg, void* const* dst, const void* const* src, const size_t* bytes);

}  // namespace kk

// kk_kernels.cu -- device kernels of the two-phase hash SpGEMM for sm_100a.
//
// Hot path (DESIGN.md Sec. 5 for the roofline of each kernel):
//   a4 k_check_compress   B -> B_C (word, mask) pairs + sortedness flags
//   a1 k_row_flops        per-row multiply-adds + symbolic work bin
//   a2/a6 k_scan_*        device exclusive scans (flops, row map)
//   a3 k_bin_*            stable row binning by work
//   a5 k_sym_warp         warp-owned shared-memory hash, accum = OR
//      k_sym_dense        CTA-owned dense bit vector over column windows
//   a7 k_num_warp         warp-owned shared hash, accum = +, fused sort
//      k_num_dense        CTA-owned dense scalar window + bitmap (sorted)
//   a8 warp bitonic sort  fused into k_num_warp's compaction
#include "kk_internal.cuh"

#include <algorithm>
#include <climits>
#include <cstdio>
#include <mutex>
#include <string>
#include <unordered_map>

namespace kk {

#define FULL 0xffffffffu

__device__ __forceinline__ unsigned lanemask_lt() {
    unsigned r;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(r));
    return r;
}
__device__ __forceinline__ unsigned lanemask_le() {
    unsigned r;
    asm("mov.u32 %0, %%lanemask_le;" : "=r"(r));
    return r;
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) v += __shfl_xor_sync(FULL, v, d);
    return v;
}

template <typename OffT>
__device__ __forceinline__ int64_t ld(const OffT* p, int64_t i) {
    return (int64_t)__ldg(p + i);
}

constexpr int ilog2(int x) { return x <= 1 ? 0 : 1 + ilog2(x >> 1); }

template <int S>
__device__ __forceinline__ uint32_t hslot(uint32_t key) {
    return (key * 0x9E3779B1u) >> (32 - ilog2(S));
}

// Claim-or-find `key` in an open-addressing table (linear probing).  Returns the slot;
// *fresh = true when this call inserted the key.  The table never overflows: the
// number of distinct keys of a row is bounded by the bin's capacity.
template <int S>
__device__ __forceinline__ uint32_t probe_claim(uint32_t* keys, uint32_t key, bool* fresh) {
    uint32_t h = hslot<S>(key);
    *fresh = false;
    while (true) {
        uint32_t cur = ((volatile uint32_t*)keys)[h];
        if (cur == key) return h;
        if (cur == EMPTY) {
            cur = atomicCAS(&keys[h], EMPTY, key);
            if (cur == EMPTY) {
                *fresh = true;
                return h;
            }
            if (cur == key) return h;
        }
        h = (h + 1) & (S - 1);
    }
}

template <int S>
__device__ __forceinline__ uint32_t probe_find(const uint32_t* keys, uint32_t key) {
    uint32_t h = hslot<S>(key);
    while (keys[h] != key) h = (h + 1) & (S - 1);
    return h;
}

// ------------------------------------------------------------------------------------
// status init
// ------------------------------------------------------------------------------------
__global__ void k_init_status(DevStatus* st) {
    if (threadIdx.x == 0) {
        st->total_flops = 0;
        st->total_words = 0;
        st->nnz_c = 0;
        st->b_sorted = 1;
        st->b_strict = 1;
        st->bad_index = 0;
        st->overflow = 0;
        st->use_comp = 0;
        st->pad = 0;
    }
    if (threadIdx.x <= NB) {
        st->sym_bin_start[threadIdx.x] = 0;
        st->num_bin_start[threadIdx.x] = 0;
    }
}

void init_status(Launch& L, DevStatus* st) {
    L.begin("init_status", L.stream);
    k_init_status<<<1, 32, 0, L.stream>>>(st);
    L.end(L.stream);
}

// ------------------------------------------------------------------------------------
// a4: sortedness check + compression of B into B_C
// One warp per row of B, 32 entries per step.  Adjacent equal words are merged with a
// segmented OR scan; a word run that crosses a 32-entry chunk is carried in registers.
// ------------------------------------------------------------------------------------
template <typename OffT>
__global__ void __launch_bounds__(256) k_check_compress(int64_t n, int64_t k, const OffT* __restrict__ brm,
                                                        const int32_t* __restrict__ bent, int do_comp,
                                                        int validate, int32_t* __restrict__ bc_len,
                                                        uint2* __restrict__ pairs, DevStatus* st) {
    const int lane = threadIdx.x & 31;
    const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    bool unsorted = false, nonstrict = false, bad = false;
    unsigned long long words = 0;
    for (int64_t j = gw; j < n; j += nw) {
        const int64_t s = ld(brm, j), e = ld(brm, j + 1);
        int prev_last = INT_MIN;
        int cw = -1;
        unsigned cm = 0;
        int outn = 0;
        for (int64_t c0 = s; c0 < e; c0 += 32) {
            const int64_t q = c0 + lane;
            const bool act = q < e;
            const int nact = (int)min((int64_t)32, e - c0);
            const int col = act ? __ldg(bent + q) : INT_MAX;
            int prev = __shfl_up_sync(FULL, col, 1);
            if (lane == 0) prev = prev_last;
            if (act) {
                unsorted |= col < prev;
                nonstrict |= col <= prev;
                bad |= (col < 0) || ((int64_t)col >= k);
            }
            prev_last = __shfl_sync(FULL, col, nact - 1);
            if (do_comp) {
                const int w = act ? (col >> 5) : INT_MAX;
                const unsigned bit = act ? (1u << (col & 31)) : 0u;
                int pw = __shfl_up_sync(FULL, w, 1);
                if (lane == 0) pw = cw;
                const bool head = act && (w != pw);
                const unsigned heads = __ballot_sync(FULL, head);
                if (cw >= 0 && (heads & 1u)) {  // the carried run ends before this chunk
                    if (lane == 0) pairs[s + outn] = make_uint2((unsigned)cw, cm);
                    ++outn;
                    cw = -1;
                    cm = 0;
                }
                const unsigned le = heads & lanemask_le();
                const int seg = le ? (31 - __clz(le)) : 0;
                unsigned v = bit;
#pragma unroll
                for (int d = 1; d < 32; d <<= 1) {
                    const unsigned t = __shfl_up_sync(FULL, v, d);
                    if (lane >= d && lane - d >= seg) v |= t;
                }
                if (!le) v |= cm;  // continuation of the carried run
                const bool flush = act && lane != nact - 1 && ((heads >> (lane + 1)) & 1u);
                const unsigned fb = __ballot_sync(FULL, flush);
                if (flush) pairs[s + outn + __popc(fb & lanemask_lt())] = make_uint2((unsigned)w, v);
                outn += __popc(fb);
                cw = __shfl_sync(FULL, w, nact - 1);
                cm = __shfl_sync(FULL, v, nact - 1);
            }
        }
        if (do_comp) {
            if (cw >= 0) {
                if (lane == 0) pairs[s + outn] = make_uint2((unsigned)cw, cm);
                ++outn;
            }
            if (lane == 0) bc_len[j] = outn;
            words += (unsigned long long)outn;
        }
    }
    if (__any_sync(FULL, unsorted) && lane == 0) atomicAnd(&st->b_sorted, 0);
    if (__any_sync(FULL, nonstrict) && lane == 0) atomicAnd(&st->b_strict, 0);
    if (validate && __any_sync(FULL, bad) && lane == 0) atomicOr(&st->bad_index, 1);
    if (do_comp && lane == 0 && words) atomicAdd(&st->total_words, words);
}

static int grid_for(int64_t warps_needed, int threads, int num_sms, int per_sm = 8) {
    int64_t blocks = (warps_needed * 32 + threads - 1) / threads;
    int64_t cap = (int64_t)num_sms * per_sm;
    if (blocks > cap) blocks = cap;
    if (blocks < 1) blocks = 1;
    return (int)blocks;
}

void check_compress(Launch& L, bool off64, const MatView& B, int64_t k, bool do_comp, bool validate,
                    int32_t* bc_len, uint2* pairs, DevStatus* st) {
    if (B.nrows == 0) return;
    const int threads = 256;
    const int grid = grid_for(B.nrows, threads, L.num_sms, 16);
    L.begin(do_comp ? "check_compress" : "check_sorted", L.stream);
    if (off64)
        k_check_compress<int64_t><<<grid, threads, 0, L.stream>>>(B.nrows, k, (const int64_t*)B.row_map, B.entries,
                                                                  do_comp, validate, bc_len, pairs, st);
    else
        k_check_compress<int32_t><<<grid, threads, 0, L.stream>>>(B.nrows, k, (const int32_t*)B.row_map, B.entries,
                                                                  do_comp, validate, bc_len, pairs, st);
    L.end(L.stream);
}

// ------------------------------------------------------------------------------------
// a1: per-row flops and the symbolic work bin of each row.
// ------------------------------------------------------------------------------------
__device__ __forceinline__ int sym_bin_of(int64_t ub) {
    if (ub <= 0) return 0;
    int b = 1;
    int64_t cap = 64;
    while (cap < ub && b < SYM_DENSE_BIN) {
        cap <<= 1;
        ++b;
    }
    return b;
}

template <typename OffT>
__global__ void __launch_bounds__(256) k_row_flops(int64_t m, int64_t n, int64_t k, const OffT* __restrict__ arm,
                                                   const int32_t* __restrict__ aent, const OffT* __restrict__ brm,
                                                   const int32_t* __restrict__ bc_len, int comp_mode, int64_t nnzB,
                                                   int validate, int64_t* __restrict__ flops,
                                                   uint8_t* __restrict__ binid, int32_t* __restrict__ counts,
                                                   DevStatus* st) {
    bool comp = false;
    if (comp_mode == 1)
        comp = true;
    else if (comp_mode == -1)
        comp = nnzB > 0 && (st->total_words * 4ull <= (unsigned long long)nnzB * 3ull);
    if (blockIdx.x == 0 && threadIdx.x == 0) st->use_comp = comp ? 1 : 0;
    const int lane = threadIdx.x & 31;
    const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int64_t kw = (k + 31) >> 5;
    unsigned long long tot = 0;
    bool bad = false;
    for (int64_t i = gw; i < m; i += nw) {
        const int64_t s = ld(arm, i), e = ld(arm, i + 1);
        int64_t f = 0, fc = 0;
        for (int64_t p = s + lane; p < e; p += 32) {
            const int j = __ldg(aent + p);
            if (validate && (j < 0 || (int64_t)j >= n)) {
                bad = true;
                continue;
            }
            f += ld(brm, (int64_t)j + 1) - ld(brm, (int64_t)j);
            if (comp) fc += __ldg(bc_len + j);
        }
        f = warp_sum(f);
        if (comp) fc = warp_sum(fc);
        if (lane == 0) {
            flops[i] = f;
            const int64_t ub = comp ? min(fc, kw) : min(f, k);
            const int b = sym_bin_of(ub);
            binid[i] = (uint8_t)b;
            if (b == 0) counts[i] = 0;
            tot += (unsigned long long)f;
        }
    }
    if (validate && __any_sync(FULL, bad) && lane == 0) atomicOr(&st->bad_index, 1);
    if (lane == 0 && tot) atomicAdd(&st->total_flops, tot);
}

void row_flops_bin(Launch& L, bool off64, const MatView& A, const MatView& B, int64_t k, int comp_mode,
                   bool validate, const int32_t* bc_len, int64_t* flops, uint8_t* binid, int32_t* counts,
                   DevStatus* st) {
    if (A.nrows == 0) return;
    const int threads = 256;
    const int grid = grid_for(A.nrows, threads, L.num_sms, 16);
    L.begin("row_flops_bin", L.stream);
    if (off64)
        k_row_flops<int64_t><<<grid, threads, 0, L.stream>>>(A.nrows, A.ncols, k, (const int64_t*)A.row_map,
                                                             A.entries, (const int64_t*)B.row_map, bc_len,
                                                             comp_mode, B.nnz, validate, flops, binid, counts, st);
    else
        k_row_flops<int32_t><<<grid, threads, 0, L.stream>>>(A.nrows, A.ncols, k, (const int32_t*)A.row_map,
                                                             A.entries, (const int32_t*)B.row_map, bc_len,
                                                             comp_mode, B.nnz, validate, flops, binid, counts, st);
    L.end(L.stream);
}

// ------------------------------------------------------------------------------------
// a2 / a6: exclusive scan (reduce -> scan partials -> downsweep), int64 accumulation.
// ------------------------------------------------------------------------------------
constexpr int SCAN_THREADS = 512;
constexpr int SCAN_ITEMS = 8;
constexpr int SCAN_TILE = SCAN_THREADS * SCAN_ITEMS;

int64_t scan_partial_len(int64_t m) { return (m + SCAN_TILE - 1) / SCAN_TILE + 2; }

// block-wide exclusive scan of one int64 per thread; returns the block total
__device__ __forceinline__ int64_t block_exclusive_scan(int64_t v, int64_t* excl) {
    __shared__ int64_t wsum[32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
    int64_t x = v;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const int64_t t = __shfl_up_sync(FULL, x, d);
        if (lane >= d) x += t;
    }
    if (lane == 31) wsum[warp] = x;
    __syncthreads();
    if (warp == 0) {
        int64_t w = lane < nwarp ? wsum[lane] : 0;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const int64_t t = __shfl_up_sync(FULL, w, d);
            if (lane >= d) w += t;
        }
        wsum[lane] = w;  // inclusive over warps
    }
    __syncthreads();
    const int64_t wbase = warp ? wsum[warp - 1] : 0;
    const int64_t total = wsum[nwarp - 1];
    *excl = wbase + x - v;
    __syncthreads();
    return total;
}

template <typename InT>
__global__ void __launch_bounds__(SCAN_THREADS) k_scan_reduce(int64_t m, const InT* __restrict__ in,
                                                              int64_t* __restrict__ partial) {
    const int64_t base = (int64_t)blockIdx.x * SCAN_TILE;
    int64_t s = 0;
#pragma unroll
    for (int t = 0; t < SCAN_ITEMS; ++t) {
        const int64_t i = base + t * SCAN_THREADS + threadIdx.x;
        if (i < m) s += (int64_t)in[i];
    }
    s = warp_sum(s);
    __shared__ int64_t ws[SCAN_THREADS / 32];
    if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x < 32) {
        int64_t v = threadIdx.x < SCAN_THREADS / 32 ? ws[threadIdx.x] : 0;
        v = warp_sum(v);
        if (threadIdx.x == 0) partial[blockIdx.x] = v;
    }
}

__global__ void __launch_bounds__(1024) k_scan_partials(int64_t nb, int64_t* __restrict__ partial,
                                                        unsigned long long* total_dst) {
    int64_t carry = 0;
    for (int64_t b0 = 0; b0 < nb; b0 += blockDim.x) {
        const int64_t b = b0 + threadIdx.x;
        const int64_t v = b < nb ? partial[b] : 0;
        int64_t ex;
        const int64_t tot = block_exclusive_scan(v, &ex);
        if (b < nb) partial[b] = carry + ex;
        carry += tot;
    }
    if (threadIdx.x == 0) {
        partial[nb] = carry;
        if (total_dst) *total_dst = (unsigned long long)carry;
    }
}

template <typename InT, typename OutT>
__global__ void __launch_bounds__(SCAN_THREADS) k_scan_down(int64_t m, const InT* __restrict__ in,
                                                            const int64_t* __restrict__ partial,
                                                            OutT* __restrict__ out, int64_t nb, int* overflow) {
    const int64_t base = (int64_t)blockIdx.x * SCAN_TILE + (int64_t)threadIdx.x * SCAN_ITEMS;
    int64_t v[SCAN_ITEMS];
    int64_t s = 0;
#pragma unroll
    for (int t = 0; t < SCAN_ITEMS; ++t) {
        const int64_t i = base + t;
        v[t] = i < m ? (int64_t)in[i] : 0;
        s += v[t];
    }
    int64_t ex;
    block_exclusive_scan(s, &ex);
    int64_t run = partial[blockIdx.x] + ex;
#pragma unroll
    for (int t = 0; t < SCAN_ITEMS; ++t) {
        const int64_t i = base + t;
        if (i < m) out[i] = (OutT)run;
        run += v[t];
    }
    if (blockIdx.x == gridDim.x - 1 && threadIdx.x == 0) {
        const int64_t total = partial[nb];
        out[m] = (OutT)total;
        if (sizeof(OutT) == 4 && total > (int64_t)INT_MAX && overflow) *overflow = 1;
    }
}

void exclusive_scan(Launch& L, bool in64, const void* in, bool out64, void* out, int64_t m, int64_t* partial,
                    unsigned long long* total_dst, int* overflow) {
    const int64_t nb = (m + SCAN_TILE - 1) / SCAN_TILE;
    if (nb == 0) {
        // m == 0: out[0] = 0, total = 0
        cudaMemsetAsync(out, 0, out64 ? 8 : 4, L.stream);
        if (total_dst) cudaMemsetAsync(total_dst, 0, 8, L.stream);
        return;
    }
    L.begin("exclusive_scan", L.stream);
    if (in64)
        k_scan_reduce<int64_t><<<(unsigned)nb, SCAN_THREADS, 0, L.stream>>>(m, (const int64_t*)in, partial);
    else
        k_scan_reduce<int32_t><<<(unsigned)nb, SCAN_THREADS, 0, L.stream>>>(m, (const int32_t*)in, partial);
    k_scan_partials<<<1, 1024, 0, L.stream>>>(nb, partial, total_dst);
    if (in64 && out64)
        k_scan_down<int64_t, int64_t><<<(unsigned)nb, SCAN_THREADS, 0, L.stream>>>(m, (const int64_t*)in, partial,
                                                                                  (int64_t*)out, nb, overflow);
    else if (in64)
        k_scan_down<int64_t, int32_t><<<(unsigned)nb, SCAN_THREADS, 0, L.stream>>>(m, (const int64_t*)in, partial,
                                                                                  (int32_t*)out, nb, overflow);
    else if (out64)
        k_scan_down<int32_t, int64_t><<<(unsigned)nb, SCAN_THREADS, 0, L.stream>>>(m, (const int32_t*)in, partial,
                                                                                  (int64_t*)out, nb, overflow);
    else
        k_scan_down<int32_t, int32_t><<<(unsigned)nb, SCAN_THREADS, 0, L.stream>>>(m, (const int32_t*)in, partial,
                                                                                  (int32_t*)out, nb, overflow);
    L.end(L.stream, 3);
}

// ------------------------------------------------------------------------------------
// a3: numeric bin ids from exact row counts, and stable binning of rows.
// ------------------------------------------------------------------------------------
__device__ __forceinline__ int num_bin_of(int64_t nnz) {
    if (nnz <= 0) return 0;
    int b = 1;
    int64_t cap = 32;
    while (cap < nnz && b < NUM_DENSE_BIN) {
        cap <<= 1;
        ++b;
    }
    return b;
}

__global__ void __launch_bounds__(256) k_numeric_binid(int64_t m, const int32_t* __restrict__ counts,
                                                       uint8_t* __restrict__ binid) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
        binid[i] = (uint8_t)num_bin_of(counts[i]);
}

void numeric_binid(Launch& L, int64_t m, const int32_t* counts, uint8_t* binid) {
    if (m == 0) return;
    int grid = (int)std::min<int64_t>((m + 255) / 256, (int64_t)L.num_sms * 16);
    L.begin("numeric_binid", L.stream);
    k_numeric_binid<<<grid, 256, 0, L.stream>>>(m, counts, binid);
    L.end(L.stream);
}

constexpr int BCHUNK = 2048;  // rows per warp in the binning passes

int64_t bin_scratch_len(int64_t m) { return ((m + BCHUNK - 1) / BCHUNK) * NB + NB + 1; }

// pass 1: per-chunk bin histogram (warp per chunk; lane b counts bin b)
__global__ void __launch_bounds__(256) k_bin_count(int64_t m, const uint8_t* __restrict__ binid,
                                                   int32_t* __restrict__ chunkcnt) {
    const int lane = threadIdx.x & 31;
    const int64_t c = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nchunks = (m + BCHUNK - 1) / BCHUNK;
    if (c >= nchunks) return;
    const int64_t r0 = c * BCHUNK, r1 = min(m, r0 + BCHUNK);
    int cnt = 0;
    for (int64_t base = r0; base < r1; base += 32) {
        const int64_t r = base + lane;
        const int b = r < r1 ? (int)binid[r] : 255;
#pragma unroll
        for (int t = 0; t < NB; ++t) {
            const unsigned bal = __ballot_sync(FULL, b == t);
            if (lane == t) cnt += __popc(bal);
        }
    }
    if (lane < NB) chunkcnt[c * NB + lane] = cnt;
}

// pass 2: per bin, exclusive scan over chunks (+ bin start); one block
__global__ void __launch_bounds__(1024) k_bin_offsets(int64_t nchunks, int32_t* __restrict__ chunkcnt,
                                                      int* __restrict__ bin_start_dst) {
    __shared__ int64_t totals[NB];
    for (int b = 0; b < NB; ++b) {
        int64_t carry = 0;
        for (int64_t c0 = 0; c0 < nchunks; c0 += blockDim.x) {
            const int64_t c = c0 + threadIdx.x;
            const int64_t v = c < nchunks ? chunkcnt[c * NB + b] : 0;
            int64_t ex;
            const int64_t tot = block_exclusive_scan(v, &ex);
            if (c < nchunks) chunkcnt[c * NB + b] = (int32_t)(carry + ex);
            carry += tot;
        }
        if (threadIdx.x == 0) totals[b] = carry;
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        int64_t run = 0;
        for (int b = 0; b < NB; ++b) {
            bin_start_dst[b] = (int)run;
            run += totals[b];
        }
        bin_start_dst[NB] = (int)run;
    }
}

// pass 3: stable scatter of rows into perm
__global__ void __launch_bounds__(256) k_bin_scatter(int64_t m, const uint8_t* __restrict__ binid,
                                                     const int32_t* __restrict__ chunkcnt,
                                                     const int* __restrict__ bin_start, int32_t* __restrict__ perm) {
    const int lane = threadIdx.x & 31;
    const int64_t c = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nchunks = (m + BCHUNK - 1) / BCHUNK;
    if (c >= nchunks) return;
    const int64_t r0 = c * BCHUNK, r1 = min(m, r0 + BCHUNK);
    int run = lane < NB ? bin_start[lane] + chunkcnt[c * NB + lane] : 0;
    for (int64_t base = r0; base < r1; base += 32) {
        const int64_t r = base + lane;
        const int b = r < r1 ? (int)binid[r] : 255;
#pragma unroll
        for (int t = 0; t < NB; ++t) {
            const unsigned bal = __ballot_sync(FULL, b == t);
            const int base_t = __shfl_sync(FULL, run, t);
            if (b == t) perm[base_t + __popc(bal & lanemask_lt())] = (int32_t)r;
            if (lane == t) run += __popc(bal);
        }
    }
}

void bin_rows(Launch& L, int64_t m, const uint8_t* binid, int32_t* scratch, int32_t* perm, int* bin_start_dst) {
    const int64_t nchunks = (m + BCHUNK - 1) / BCHUNK;
    if (nchunks == 0) {
        cudaMemsetAsync(bin_start_dst, 0, sizeof(int) * (NB + 1), L.stream);
        return;
    }
    const int grid = (int)((nchunks * 32 + 255) / 256);
    L.begin("bin_rows", L.stream);
    k_bin_count<<<grid, 256, 0, L.stream>>>(m, binid, scratch);
    k_bin_offsets<<<1, 1024, 0, L.stream>>>(nchunks, scratch, bin_start_dst);
    k_bin_scatter<<<grid, 256, 0, L.stream>>>(m, binid, scratch, bin_start_dst, perm);
    L.end(L.stream, 3);
}

// ------------------------------------------------------------------------------------
// a5: symbolic, warp-owned shared hash ("HashmapAccumulator"; accum = OR
// with compression, set insert without).  Each warp owns one row at a time; G lanes
// walk one B row, 32/G rows of B in flight per step ("entries in each
// referenced row of B are processed using vector parallelism").
// ------------------------------------------------------------------------------------
template <typename OffT, int S>
__global__ void __launch_bounds__(256) k_sym_warp(const OffT* __restrict__ arm, const int32_t* __restrict__ aent,
                                                  const OffT* __restrict__ brm, const int32_t* __restrict__ bent,
                                                  const int32_t* __restrict__ bc_len, const uint2* __restrict__ pairs,
                                                  const int32_t* __restrict__ perm, const int* __restrict__ bin_start,
                                                  int bin, int logG, int32_t* __restrict__ counts,
                                                  const DevStatus* __restrict__ st) {
    extern __shared__ uint32_t sm_sym[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, warps = blockDim.x >> 5;
    uint32_t* keys = sm_sym + (size_t)warp * 2 * S;
    uint32_t* masks = keys + S;
    const int r0 = bin_start[bin], r1 = bin_start[bin + 1];
    if (r0 + blockIdx.x * warps + warp >= r1) return;
    for (int t = lane; t < S; t += 32) {
        keys[t] = EMPTY;
        masks[t] = 0;
    }
    __syncwarp();
    const bool comp = st->use_comp != 0;
    const int G = 1 << logG, per = 32 >> logG, gl = lane & (G - 1), sub = lane >> logG;
    for (int r = r0 + blockIdx.x * warps + warp; r < r1; r += gridDim.x * warps) {
        const int i = perm[r];
        const int64_t s = ld(arm, i), e = ld(arm, i + 1);
        int cnt = 0;
        for (int64_t p0 = s; p0 < e; p0 += per) {
            const int64_t p = p0 + sub;
            if (p < e) {
                const int j = __ldg(aent + p);
                const int64_t bs = ld(brm, j);
                bool fresh;
                if (comp) {
                    const int64_t be = bs + __ldg(bc_len + j);
                    for (int64_t q = bs + gl; q < be; q += G) {
                        const uint2 pr = __ldg(pairs + q);
                        const uint32_t h = probe_claim<S>(keys, pr.x, &fresh);
                        atomicOr(&masks[h], pr.y);
                    }
                } else {
                    const int64_t be = ld(brm, j + 1);
                    for (int64_t q = bs + gl; q < be; q += G) {
                        probe_claim<S>(keys, (uint32_t)__ldg(bent + q), &fresh);
                        cnt += fresh;
                    }
                }
            }
        }
        __syncwarp();
        for (int t = lane; t < S; t += 32) {
            if (keys[t] != EMPTY) {
                if (comp) cnt += __popc(masks[t]);
                keys[t] = EMPTY;
                masks[t] = 0;
            }
        }
        cnt = warp_sum(cnt);
        if (lane == 0) counts[i] = cnt;
        __syncwarp();
    }
}

// Walk the part of a SORTED row [q0, qe) whose keys are below `hi`, 32 entries per step;
// calls f(q) for each such entry, returns the first position not processed.
template <typename KeyF, typename F>
__device__ __forceinline__ int64_t walk_sorted(int64_t q0, int64_t qe, int64_t hi, KeyF key, F f) {
    const int lane = threadIdx.x & 31;
    while (q0 < qe) {
        const int64_t q = q0 + lane;
        const int64_t kq = q < qe ? key(q) : INT64_MAX;
        const bool in = kq < hi;
        if (in) f(q, kq);
        const unsigned bal = __ballot_sync(FULL, in);
        q0 += __popc(bal);
        if (bal != FULL) break;
    }
    return q0;
}

template <typename T>
__device__ __forceinline__ T block_sum(T v) {
    __shared__ T red[32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    v = warp_sum(v);
    __syncthreads();
    if (lane == 0) red[warp] = v;
    __syncthreads();
    T t = 0;
    for (int w = 0; w < nw; ++w) t += red[w];
    return t;
}

// a5 for rows whose bound exceeds the warp tables: the paper's dense bit-vector
// accumulator in one CTA's shared memory, over windows of `wbits`
// columns when k is larger.  Sorted B rows are resumed from per-entry cursors.
template <typename OffT>
__global__ void __launch_bounds__(512) k_sym_dense(const OffT* __restrict__ arm, const int32_t* __restrict__ aent,
                                                   const OffT* __restrict__ brm, const int32_t* __restrict__ bent,
                                                   const int32_t* __restrict__ bc_len,
                                                   const uint2* __restrict__ pairs, const int32_t* __restrict__ perm,
                                                   const int* __restrict__ bin_start, int bin, int64_t k,
                                                   int64_t wbits, int32_t* __restrict__ cursors,
                                                   int32_t* __restrict__ counts, const DevStatus* __restrict__ st) {
    extern __shared__ uint32_t bmp[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, warps = blockDim.x >> 5;
    const int r0 = bin_start[bin], r1 = bin_start[bin + 1];
    if (r0 + (int)blockIdx.x >= r1) return;
    const int64_t maxw = wbits >> 5;
    for (int64_t t = threadIdx.x; t < maxw; t += blockDim.x) bmp[t] = 0;
    __syncthreads();
    const bool comp = st->use_comp != 0;
    const bool sorted = st->b_sorted != 0;
    for (int r = r0 + blockIdx.x; r < r1; r += gridDim.x) {
        const int i = perm[r];
        const int64_t s = ld(arm, i), e = ld(arm, i + 1);
        long long cnt = 0;
        for (int64_t lo = 0; lo < k; lo += wbits) {
            const int64_t hi = min(k, lo + wbits);
            const bool single = (lo == 0 && hi == k);
            const int64_t low = lo >> 5, hiw = (hi + 31) >> 5;
            for (int64_t p = s + warp; p < e; p += warps) {
                const int j = __ldg(aent + p);
                const int64_t bs = ld(brm, j);
                if (comp) {
                    const int64_t be = bs + __ldg(bc_len + j);
                    if (single) {
                        for (int64_t q = bs + lane; q < be; q += 32) {
                            const uint2 pr = __ldg(pairs + q);
                            atomicOr(&bmp[pr.x], pr.y);
                        }
                    } else if (sorted) {
                        const int64_t q0 = bs + (lo == 0 ? 0 : cursors[p]);
                        const int64_t qn = walk_sorted(
                            q0, be, hiw, [&](int64_t q) { return (int64_t)__ldg(&pairs[q].x); },
                            [&](int64_t q, int64_t w) { atomicOr(&bmp[w - low], __ldg(&pairs[q].y)); });
                        if (lane == 0) cursors[p] = (int32_t)(qn - bs);
                    } else {
                        for (int64_t q = bs + lane; q < be; q += 32) {
                            const uint2 pr = __ldg(pairs + q);
                            if ((int64_t)pr.x >= low && (int64_t)pr.x < hiw) atomicOr(&bmp[pr.x - low], pr.y);
                        }
                    }
                } else {
                    const int64_t be = ld(brm, j + 1);
                    if (single) {
                        for (int64_t q = bs + lane; q < be; q += 32) {
                            const int c = __ldg(bent + q);
                            atomicOr(&bmp[c >> 5], 1u << (c & 31));
                        }
                    } else if (sorted) {
                        const int64_t q0 = bs + (lo == 0 ? 0 : cursors[p]);
                        const int64_t qn = walk_sorted(
                            q0, be, hi, [&](int64_t q) { return (int64_t)__ldg(bent + q); },
                            [&](int64_t q, int64_t c) { atomicOr(&bmp[(c - lo) >> 5], 1u << (c & 31)); });
                        if (lane == 0) cursors[p] = (int32_t)(qn - bs);
                    } else {
                        for (int64_t q = bs + lane; q < be; q += 32) {
                            const int c = __ldg(bent + q);
                            if (c >= lo && c < hi) atomicOr(&bmp[(c - lo) >> 5], 1u << (c & 31));
                        }
                    }
                }
            }
            __syncthreads();
            const int64_t nw = hiw - low;
            for (int64_t t = threadIdx.x; t < nw; t += blockDim.x) {
                const uint32_t v = bmp[t];
                if (v) {
                    cnt += __popc(v);
                    bmp[t] = 0;
                }
            }
            __syncthreads();
        }
        cnt = block_sum(cnt);
        if (threadIdx.x == 0) counts[i] = (int32_t)cnt;
    }
}

// ------------------------------------------------------------------------------------
// launch configuration helpers
// ------------------------------------------------------------------------------------
struct KCfg {
    int threads;
    size_t smem;
    int grid_cap;  // max resident CTAs on the device
};

static std::mutex g_cfg_mu;
static std::unordered_map<const void*, KCfg> g_cfg;

template <typename K>
static KCfg kernel_cfg(K kern, int threads, size_t smem, int num_sms) {
    std::lock_guard<std::mutex> lk(g_cfg_mu);
    auto it = g_cfg.find((const void*)kern);
    if (it != g_cfg.end() && it->second.threads == threads && it->second.smem == smem) return it->second;
    if (smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem);
    if (per_sm < 1) per_sm = 1;
    KCfg c{threads, smem, per_sm * num_sms};
    g_cfg[(const void*)kern] = c;
    return c;
}

// stable names for the timing table: "<base>_S<slots>"
static const char* kname(const char* base, int S) {
    static std::mutex mu;
    static std::unordered_map<std::string, std::string> names;
    std::lock_guard<std::mutex> lk(mu);
    std::string key = std::string(base) + "_S" + std::to_string(S);
    auto it = names.find(key);
    if (it == names.end()) it = names.emplace(key, key).first;
    return it->second.c_str();
}

static int sym_warps_for(int S) { return S <= 512 ? 8 : (S == 1024 ? 4 : (S == 2048 ? 2 : 1)); }

template <typename OffT, int S>
static void launch_sym_warp(Launch& L, const SymArgs& a, int bin) {
    const int warps = sym_warps_for(S);
    const size_t smem = (size_t)warps * 2 * S * sizeof(uint32_t);
    auto kern = k_sym_warp<OffT, S>;
    KCfg c = kernel_cfg(kern, warps * 32, smem, L.num_sms);
    int grid = c.grid_cap;
    int64_t need = (a.A.nrows + warps - 1) / warps;
    if (need < grid) grid = (int)(need > 0 ? need : 1);
    L.begin(kname("sym_warp", S), L.stream);
    kern<<<grid, warps * 32, smem, L.stream>>>((const OffT*)a.A.row_map, a.A.entries, (const OffT*)a.B.row_map,
                                               a.B.entries, a.bc_len, a.pairs, a.perm, a.bin_start, bin, a.logG,
                                               a.counts, a.st);
    L.end(L.stream);
}

template <typename OffT>
static void symbolic_bins_t(Launch& L, const SymArgs& a, cudaStream_t dense_stream) {
    // dense rows first (heaviest), on their own stream when given
    {
        const int threads = 512;
        int64_t wbits = 200 * 1024 * 8;  // 200 KB bit vector
        const int64_t k32 = ((a.k + 31) / 32) * 32;
        if (k32 < wbits) wbits = k32 > 0 ? k32 : 32;
        const size_t smem = (size_t)(wbits / 8);
        auto kern = k_sym_dense<OffT>;
        KCfg c = kernel_cfg(kern, threads, smem, L.num_sms);
        cudaStream_t s = dense_stream ? dense_stream : L.stream;
        L.begin("sym_dense", s);
        kern<<<c.grid_cap, threads, smem, s>>>((const OffT*)a.A.row_map, a.A.entries, (const OffT*)a.B.row_map,
                                               a.B.entries, a.bc_len, a.pairs, a.perm, a.bin_start, SYM_DENSE_BIN,
                                               a.k, wbits, a.cursors, a.counts, a.st);
        L.end(s);
    }
    launch_sym_warp<OffT, 4096>(L, a, 7);
    launch_sym_warp<OffT, 2048>(L, a, 6);
    launch_sym_warp<OffT, 1024>(L, a, 5);
    launch_sym_warp<OffT, 512>(L, a, 4);
    launch_sym_warp<OffT, 256>(L, a, 3);
    launch_sym_warp<OffT, 128>(L, a, 2);
    launch_sym_warp<OffT, 64>(L, a, 1);
}

void symbolic_bins(Launch& L, const SymArgs& a, cudaStream_t dense_stream) {
    if (a.A.nrows == 0) return;
    if (a.off64)
        symbolic_bins_t<int64_t>(L, a, dense_stream);
    else
        symbolic_bins_t<int32_t>(L, a, dense_stream);
}

// ------------------------------------------------------------------------------------
// a8: warp bitonic sort of 32*E keys held E per lane (element e = lane*E + r)
// (team-level bitonic sort, mapped to one warp's registers)
// ------------------------------------------------------------------------------------
template <int E>
__device__ __forceinline__ void warp_bitonic_sort(uint32_t (&v)[E]) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int k = 2; k <= 32 * E; k <<= 1) {
#pragma unroll
        for (int j = k >> 1; j > 0; j >>= 1) {
            if (j >= E) {
                const int lj = j / E;
#pragma unroll
                for (int r = 0; r < E; ++r) {
                    const int e = lane * E + r;
                    const uint32_t o = __shfl_xor_sync(FULL, v[r], lj);
                    const bool up = (e & k) == 0;
                    const bool lower = (e & j) == 0;
                    v[r] = (up == lower) ? min(v[r], o) : max(v[r], o);
                }
            } else {
#pragma unroll
                for (int r = 0; r < E; ++r) {
                    const int pr = r ^ j;
                    if (pr > r) {
                        const int e = lane * E + r;
                        const bool up = (e & k) == 0;
                        const uint32_t x = v[r], y = v[pr];
                        const bool sw = up ? (x > y) : (x < y);
                        v[r] = sw ? y : x;
                        v[pr] = sw ? x : y;
                    }
                }
            }
        }
    }
}

// ------------------------------------------------------------------------------------
// a7: numeric, warp-owned shared hash (accum = +).  With G = 32
// lanes on one strictly increasing B row the keys of a step are distinct, so values
// are updated with plain shared loads/stores; otherwise with shared atomicAdd.
// The compaction is followed by the fused per-row sort (a8) and a coalesced write.
// ------------------------------------------------------------------------------------
template <typename OffT, typename ValT, int S, bool SORT>
__global__ void __launch_bounds__(256) k_num_warp(const OffT* __restrict__ arm, const int32_t* __restrict__ aent,
                                                  const ValT* __restrict__ aval, const OffT* __restrict__ brm,
                                                  const int32_t* __restrict__ bent, const ValT* __restrict__ bval,
                                                  const OffT* __restrict__ crm, int32_t* __restrict__ cent,
                                                  ValT* __restrict__ cval, const int32_t* __restrict__ perm,
                                                  const int* __restrict__ bin_start, int bin, int logG,
                                                  const DevStatus* __restrict__ st) {
    extern __shared__ __align__(16) unsigned char sm_num[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, warps = blockDim.x >> 5;
    constexpr size_t WB = (size_t)S * sizeof(ValT) + (size_t)S * 4 + (size_t)S * 2;
    ValT* vals = (ValT*)(sm_num + (size_t)warp * WB);
    uint32_t* keys = (uint32_t*)(vals + S);
    uint32_t* stage = keys + S;
    const int r0 = bin_start[bin], r1 = bin_start[bin + 1];
    if (r0 + blockIdx.x * warps + warp >= r1) return;
    for (int t = lane; t < S; t += 32) {
        keys[t] = EMPTY;
        vals[t] = (ValT)0;
    }
    __syncwarp();
    const bool plain = (logG == 5) && (st->b_strict != 0);
    const int G = 1 << logG, per = 32 >> logG, gl = lane & (G - 1), sub = lane >> logG;
    for (int r = r0 + blockIdx.x * warps + warp; r < r1; r += gridDim.x * warps) {
        const int i = perm[r];
        const int64_t s = ld(arm, i), e = ld(arm, i + 1);
        const int64_t cb = ld(crm, i);
        const int clen = (int)(ld(crm, i + 1) - cb);
        for (int64_t p0 = s; p0 < e; p0 += per) {
            const int64_t p = p0 + sub;
            if (p < e) {
                const int j = __ldg(aent + p);
                const ValT a = __ldg(aval + p);
                const int64_t bs = ld(brm, j), be = ld(brm, j + 1);
                bool fresh;
                for (int64_t q = bs + gl; q < be; q += G) {
                    const uint32_t col = (uint32_t)__ldg(bent + q);
                    const ValT prod = a * __ldg(bval + q);
                    const uint32_t h = probe_claim<S>(keys, col, &fresh);
                    if (plain)
                        vals[h] += prod;
                    else
                        atomicAdd(&vals[h], prod);
                }
            }
            if (plain) __syncwarp();
        }
        __syncwarp();
        // compaction (slot order) into stage: keys when sorting, slots otherwise
        int n = 0;
#pragma unroll 4
        for (int c = 0; c < S; c += 32) {
            const uint32_t kk = keys[c + lane];
            const bool occ = kk != EMPTY;
            const unsigned bal = __ballot_sync(FULL, occ);
            if (occ) stage[n + __popc(bal & lanemask_lt())] = SORT ? kk : (uint32_t)(c + lane);
            n += __popc(bal);
        }
        __syncwarp();
        if (n > clen) n = clen;  // guard: never write past the row (row map from another product)
        if (SORT) {
            constexpr int E = S / 64;
            uint32_t v[E];
#pragma unroll
            for (int r2 = 0; r2 < E; ++r2) {
                const int idx = lane * E + r2;
                v[r2] = idx < n ? stage[idx] : EMPTY;
            }
            warp_bitonic_sort<E>(v);
            __syncwarp();
#pragma unroll
            for (int r2 = 0; r2 < E; ++r2) {
                const int idx = lane * E + r2;
                if (idx < n) stage[idx] = v[r2];
            }
            __syncwarp();
            for (int t = lane; t < n; t += 32) {
                const uint32_t col = stage[t];
                const uint32_t h = probe_find<S>(keys, col);
                cent[cb + t] = (int32_t)col;
                cval[cb + t] = vals[h];
            }
        } else {
            for (int t = lane; t < n; t += 32) {
                const uint32_t h = stage[t];
                cent[cb + t] = (int32_t)keys[h];
                cval[cb + t] = vals[h];
            }
        }
        __syncwarp();
        for (int t = lane; t < S; t += 32) {
            keys[t] = EMPTY;
            vals[t] = (ValT)0;
        }
        __syncwarp();
    }
}

// a7 for rows above the warp tables: column-windowed dense scalar accumulator (the
// paper's dense numeric accumulator, held per CTA in shared memory
// instead of per thread) with a presence bitmap; compaction walks the bitmap in
// column order, so the output row is sorted without a sort.
template <typename OffT, typename ValT>
__global__ void __launch_bounds__(256) k_num_dense(const OffT* __restrict__ arm, const int32_t* __restrict__ aent,
                                                   const ValT* __restrict__ aval, const OffT* __restrict__ brm,
                                                   const int32_t* __restrict__ bent, const ValT* __restrict__ bval,
                                                   const OffT* __restrict__ crm, int32_t* __restrict__ cent,
                                                   ValT* __restrict__ cval, const int32_t* __restrict__ perm,
                                                   const int* __restrict__ bin_start, int bin, int64_t k, int W,
                                                   int32_t* __restrict__ cursors, const DevStatus* __restrict__ st) {
    extern __shared__ __align__(16) unsigned char sm_dense[];
    ValT* win = (ValT*)sm_dense;
    uint32_t* bmp = (uint32_t*)(win + W);
    __shared__ int wcnt[8];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, warps = blockDim.x >> 5;
    const int r0 = bin_start[bin], r1 = bin_start[bin + 1];
    if (r0 + (int)blockIdx.x >= r1) return;
    for (int t = threadIdx.x; t < W; t += blockDim.x) win[t] = (ValT)0;
    for (int t = threadIdx.x; t < (W >> 5); t += blockDim.x) bmp[t] = 0;
    __syncthreads();
    const bool sorted = st->b_sorted != 0;
    for (int r = r0 + blockIdx.x; r < r1; r += gridDim.x) {
        const int i = perm[r];
        const int64_t s = ld(arm, i), e = ld(arm, i + 1);
        const int64_t cb = ld(crm, i);
        const int64_t clen = ld(crm, i + 1) - cb;
        int64_t outpos = 0;
        for (int64_t lo = 0; lo < k; lo += W) {
            const int64_t hi = min(k, lo + (int64_t)W);
            const bool single = (lo == 0 && hi == k);
            for (int64_t p = s + warp; p < e; p += warps) {
                const int j = __ldg(aent + p);
                const ValT a = __ldg(aval + p);
                const int64_t bs = ld(brm, j), be = ld(brm, j + 1);
                auto ins = [&](int64_t q, int64_t c) {
                    const int x = (int)(c - lo);
                    atomicAdd(&win[x], a * __ldg(bval + q));
                    atomicOr(&bmp[x >> 5], 1u << (x & 31));
                };
                if (single) {
                    for (int64_t q = bs + lane; q < be; q += 32) ins(q, __ldg(bent + q));
                } else if (sorted) {
                    const int64_t q0 = bs + (lo == 0 ? 0 : cursors[p]);
                    const int64_t qn = walk_sorted(
                        q0, be, hi, [&](int64_t q) { return (int64_t)__ldg(bent + q); }, ins);
                    if (lane == 0) cursors[p] = (int32_t)(qn - bs);
                } else {
                    for (int64_t q = bs + lane; q < be; q += 32) {
                        const int c = __ldg(bent + q);
                        if (c >= lo && c < hi) ins(q, c);
                    }
                }
            }
            __syncthreads();
            // compaction in column order: warp w owns words [w0, w1)
            const int nw = (int)((hi - lo + 31) >> 5);
            const int w0 = (int)((int64_t)warp * nw / warps), w1 = (int)((int64_t)(warp + 1) * nw / warps);
            int c = 0;
            for (int t = w0 + lane; t < w1; t += 32) c += __popc(bmp[t]);
            c = warp_sum(c);
            if (lane == 0) wcnt[warp] = c;
            __syncthreads();
            int off = 0, tot = 0;
            for (int w = 0; w < warps; ++w) {
                if (w < warp) off += wcnt[w];
                tot += wcnt[w];
            }
            for (int t0 = w0; t0 < w1; t0 += 32) {
                const int t = t0 + lane;
                const uint32_t wv = t < w1 ? bmp[t] : 0u;
                unsigned nz = __ballot_sync(FULL, wv != 0);
                while (nz) {
                    const int src = __ffs(nz) - 1;
                    nz &= nz - 1;
                    const uint32_t word = __shfl_sync(FULL, wv, src);
                    const int tw = t0 + src;
                    if ((word >> lane) & 1u) {
                        const int64_t pos = outpos + off + __popc(word & lanemask_lt());
                        const int x = tw * 32 + lane;
                        if (pos < clen) {
                            cent[cb + pos] = (int32_t)(lo + x);
                            cval[cb + pos] = win[x];
                        }
                        win[x] = (ValT)0;
                    }
                    off += __popc(word);
                }
                if (t < w1 && wv) bmp[t] = 0;
            }
            outpos += tot;
            __syncthreads();
        }
    }
}

template <typename OffT, typename ValT, int S, bool SORT>
static void launch_num_warp(Launch& L, const NumArgs& a, int bin) {
    const int rows = a.host_bin_start[bin + 1] - a.host_bin_start[bin];
    if (rows <= 0) return;
    const int warps = (S <= 256) ? 8 : 4;
    const size_t smem = (size_t)warps * ((size_t)S * sizeof(ValT) + (size_t)S * 6);
    auto kern = k_num_warp<OffT, ValT, S, SORT>;
    KCfg c = kernel_cfg(kern, warps * 32, smem, L.num_sms);
    int64_t need = (rows + warps - 1) / warps;
    int grid = (int)std::min<int64_t>(need, c.grid_cap);
    L.begin(kname("num_warp", S), L.stream);
    kern<<<grid, warps * 32, smem, L.stream>>>((const OffT*)a.A.row_map, a.A.entries, (const ValT*)a.A.values,
                                               (const OffT*)a.B.row_map, a.B.entries, (const ValT*)a.B.values,
                                               (const OffT*)a.c_row_map, a.c_entries, (ValT*)a.c_values, a.perm,
                                               a.bin_start, bin, a.logG, a.st);
    L.end(L.stream);
}

template <typename OffT, typename ValT, bool SORT>
static void numeric_bins_t(Launch& L, const NumArgs& a, cudaStream_t dense_stream) {
    const int drows = a.host_bin_start[NUM_DENSE_BIN + 1] - a.host_bin_start[NUM_DENSE_BIN];
    if (drows > 0) {
        const int threads = 256;
        const size_t budget = 200 * 1024;
        int64_t W = (int64_t)(budget / (sizeof(ValT) + 0.125)) & ~31ll;
        const int64_t k32 = ((a.k + 31) / 32) * 32;
        if (k32 < W) W = k32 > 0 ? k32 : 32;
        const size_t smem = (size_t)W * sizeof(ValT) + (size_t)(W / 32) * 4;
        auto kern = k_num_dense<OffT, ValT>;
        KCfg c = kernel_cfg(kern, threads, smem, L.num_sms);
        const int grid = (int)std::min<int64_t>(drows, c.grid_cap);
        cudaStream_t s = dense_stream ? dense_stream : L.stream;
        L.begin("num_dense", s);
        kern<<<grid, threads, smem, s>>>((const OffT*)a.A.row_map, a.A.entries, (const ValT*)a.A.values,
                                         (const OffT*)a.B.row_map, a.B.entries, (const ValT*)a.B.values,
                                         (const OffT*)a.c_row_map, a.c_entries, (ValT*)a.c_values, a.perm, a.bin_start,
                                         NUM_DENSE_BIN, a.k, (int)W, a.cursors, a.st);
        L.end(s);
    }
    launch_num_warp<OffT, ValT, 1024, SORT>(L, a, 5);
    launch_num_warp<OffT, ValT, 512, SORT>(L, a, 4);
    launch_num_warp<OffT, ValT, 256, SORT>(L, a, 3);
    launch_num_warp<OffT, ValT, 128, SORT>(L, a, 2);
    launch_num_warp<OffT, ValT, 64, SORT>(L, a, 1);
}

void numeric_bins(Launch& L, const NumArgs& a, cudaStream_t dense_stream) {
    if (a.A.nrows == 0) return;
    if (a.off64) {
        if (a.f64) {
            if (a.sort) numeric_bins_t<int64_t, double, true>(L, a, dense_stream);
            else numeric_bins_t<int64_t, double, false>(L, a, dense_stream);
        } else {
            if (a.sort) numeric_bins_t<int64_t, float, true>(L, a, dense_stream);
            else numeric_bins_t<int64_t, float, false>(L, a, dense_stream);
        }
    } else {
        if (a.f64) {
            if (a.sort) numeric_bins_t<int32_t, double, true>(L, a, dense_stream);
            else numeric_bins_t<int32_t, double, false>(L, a, dense_stream);
        } else {
            if (a.sort) numeric_bins_t<int32_t, float, true>(L, a, dense_stream);
            else numeric_bins_t<int32_t, float, false>(L, a, dense_stream);
        }
    }
}

}  // namespace kk

// kk_setup.cu -- a1-a4, a6: status block, B check/compression, row flops + bins, scans, binning.
//
//   a4 k_check_compress   B -> B_C (word, mask) pairs + sortedness flags
//   a1 k_row_flops        per-row multiply-adds + symbolic work bin
//   a2/a6 k_scan_*        device exclusive scans (flops, row map)
//   a3 k_bin_*            stable row binning by work
#include "kk_device.cuh"

#include <algorithm>
#include <atomic>
#include <chrono>

namespace kk {
// ------------------------------------------------------------------------------------
// status init
// ------------------------------------------------------------------------------------
__global__ void k_init_status(DevStatus* st, StatusCarry c) {
    if (threadIdx.x == 0) {
        st->total_flops = 0;
        st->total_words = c.total_words;
        st->nnz_c = 0;
        st->pat_used = 0;
        st->b_sorted = c.b_sorted;
        st->b_strict = c.b_strict;
        st->bad_index = c.bad_index;
        st->overflow = 0;
        st->use_comp = 0;
        st->pad = 0;
    }
    if (threadIdx.x <= NB) {
        st->sym_bin_start[threadIdx.x] = 0;
        st->num_bin_start[threadIdx.x] = 0;
    }
}

// p[0..n) += delta (the host-buffer product rebases a row block's row map to global offsets on
// the device before copying it out)
template <typename T>
__global__ void __launch_bounds__(256) k_add_offset(T* __restrict__ p, int64_t n, T delta, T* __restrict__ out) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const T v = p[i] + delta;
        if (out)
            out[i] = v;
        else
            p[i] = v;
    }
}

void add_offset(Launch& L, bool off64, void* p, int64_t n, int64_t delta, void* out) {
    if (n <= 0 || (delta == 0 && !out)) return;
    const int grid = (int)std::min<int64_t>((n + 255) / 256, (int64_t)L.num_sms * 8);
    L.begin("add_offset", L.stream);
    if (off64)
        k_add_offset<int64_t><<<grid, 256, 0, L.stream>>>((int64_t*)p, n, (int64_t)delta, (int64_t*)out);
    else
        k_add_offset<int32_t><<<grid, 256, 0, L.stream>>>((int32_t*)p, n, (int32_t)delta, (int32_t*)out);
    L.end(L.stream);
}

// Status words to the host by SM stores into mapped pinned memory: the read does not queue on
// a copy engine, so a bulk device->host copy in flight on another stream (the host-buffer
// product's pipeline) cannot delay the phase's sync behind it.
struct WordSegs {
    uint32_t* dst[4];
    const uint32_t* src[4];
    int n[4];
};

__global__ void __launch_bounds__(256) k_post_words(WordSegs w, int nseg) {
    for (int g = 0; g < nseg; ++g)
        for (int i = threadIdx.x; i < w.n[g]; i += blockDim.x) w.dst[g][i] = w.src[g][i];
}

void post_words(Launch& L, int nseg, void* const* dst, const void* const* src, const size_t* bytes) {
    WordSegs w{};
    for (int g = 0; g < nseg; ++g) {
        w.dst[g] = (uint32_t*)dst[g];
        w.src[g] = (const uint32_t*)src[g];
        w.n[g] = (int)(bytes[g] / 4);
    }
    L.begin("post_status", L.stream);
    k_post_words<<<1, 256, 0, L.stream>>>(w, nseg);
    L.end(L.stream);
}

// dst[i] = src[i] - base, i < n (a row block's row map rebased to 0; dst may be src)
template <typename T>
__global__ void __launch_bounds__(256) k_rebase(T* dst, const T* src, int64_t n, T base) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        dst[i] = src[i] - base;
}

void rebase_row_map(Launch& L, bool off64, void* dst, const void* src, int64_t n, int64_t base) {
    if (n <= 0) return;
    const int grid = (int)std::min<int64_t>((n + 255) / 256, (int64_t)L.num_sms * 8);
    L.begin("rebase_row_map", L.stream);
    if (off64)
        k_rebase<int64_t><<<grid, 256, 0, L.stream>>>((int64_t*)dst, (const int64_t*)src, n, (int64_t)base);
    else
        k_rebase<int32_t><<<grid, 256, 0, L.stream>>>((int32_t*)dst, (const int32_t*)src, n, (int32_t)base);
    L.end(L.stream);
}

// a row block of a matrix already on the device, in one launch: row map rebased by `base`,
// entries and values copied (16-byte words when aligned)
template <typename T>
__global__ void __launch_bounds__(256) k_copy_rows(T* __restrict__ rm_dst, const T* __restrict__ rm_src, int64_t nrm,
                                                   T base, char* __restrict__ e_dst, const char* __restrict__ e_src,
                                                   int64_t e_bytes, char* __restrict__ v_dst,
                                                   const char* __restrict__ v_src, int64_t v_bytes) {
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, nt = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = tid; i < nrm; i += nt) rm_dst[i] = rm_src[i] - base;
    auto copy = [&](char* d, const char* sp, int64_t bytes) {
        if ((((uintptr_t)d | (uintptr_t)sp) & 15) == 0) {
            const int64_t n16 = bytes >> 4;
            for (int64_t i = tid; i < n16; i += nt) ((int4*)d)[i] = __ldg((const int4*)sp + i);
            for (int64_t i = (n16 << 4) + tid; i < bytes; i += nt) d[i] = sp[i];
        } else {
            for (int64_t i = tid; i < bytes; i += nt) d[i] = sp[i];
        }
    };
    copy(e_dst, e_src, e_bytes);
    copy(v_dst, v_src, v_bytes);
}

void copy_rows(Launch& L, bool off64, void* rm_dst, const void* rm_src, int64_t nrm, int64_t base, void* e_dst,
               const void* e_src, int64_t e_bytes, void* v_dst, const void* v_src, int64_t v_bytes) {
    const int64_t work = std::max<int64_t>(nrm, std::max(e_bytes, v_bytes) / 16);
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((work + 255) / 256, (int64_t)L.num_sms * 8));
    L.begin("copy_rows", L.stream);
    if (off64)
        k_copy_rows<int64_t><<<grid, 256, 0, L.stream>>>((int64_t*)rm_dst, (const int64_t*)rm_src, nrm, (int64_t)base,
                                                         (char*)e_dst, (const char*)e_src, e_bytes, (char*)v_dst,
                                                         (const char*)v_src, v_bytes);
    else
        k_copy_rows<int32_t><<<grid, 256, 0, L.stream>>>((int32_t*)rm_dst, (const int32_t*)rm_src, nrm, (int32_t)base,
                                                         (char*)e_dst, (const char*)e_src, e_bytes, (char*)v_dst,
                                                         (const char*)v_src, v_bytes);
    L.end(L.stream);
}

void init_status(Launch& L, DevStatus* st, const StatusCarry* carry) {
    L.begin("init_status", L.stream);
    k_init_status<<<1, 32, 0, L.stream>>>(st, carry ? *carry : StatusCarry());
    L.end(L.stream);
}

// ------------------------------------------------------------------------------------
// a4: sortedness check + compression of B into B_C
// A warp takes 32 consecutive rows of B; each lane scans its own row sequentially (B
// rows are short on stencil and graph inputs), merging adjacent equal words.  Rows
// longer than LANE_ROW_MAX are then walked by the whole warp, 32 entries per step, with
// a segmented OR scan; a word run that crosses a 32-entry chunk is carried in registers.
// Per row it also writes bmeta = {nnz, |B_C row|, first column, last column}, the
// record a1 gathers once per A entry.
// ------------------------------------------------------------------------------------
constexpr int LANE_ROW_MAX = 64;

struct CompressFlags {
    bool unsorted = false, nonstrict = false, bad = false;
    unsigned long long words = 0;
};

template <typename OffT>
__device__ __forceinline__ void compress_row_warp(int64_t j, int64_t k, const OffT* __restrict__ brm,
                                                  const int32_t* __restrict__ bent, bool do_comp,
                                                  int32_t* __restrict__ bc_len, uint2* __restrict__ pairs,
                                                  int4* __restrict__ bmeta, CompressFlags& fl) {
    const int lane = threadIdx.x & 31;
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
            fl.unsorted |= col < prev;
            fl.nonstrict |= col <= prev;
            fl.bad |= (col < 0) || ((int64_t)col >= k);
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
    if (do_comp && cw >= 0) {
        if (lane == 0) pairs[s + outn] = make_uint2((unsigned)cw, cm);
        ++outn;
    }
    if (lane == 0) {
        if (do_comp) bc_len[j] = outn;
        if (bmeta) bmeta[j] = make_int4((int)(e - s), do_comp ? outn : 0, s < e ? __ldg(bent + s) : INT_MAX,
                                        s < e ? prev_last : -1);
    }
    if (lane == 0 && do_comp) fl.words += (unsigned long long)outn;
}

template <typename OffT>
__global__ void __launch_bounds__(256) k_check_compress(int64_t n, int64_t k, const OffT* __restrict__ brm,
                                                        const int32_t* __restrict__ bent, int do_comp,
                                                        int validate, int32_t* __restrict__ bc_len,
                                                        uint2* __restrict__ pairs, int4* __restrict__ bmeta,
                                                        DevStatus* st, int lane_max, int64_t row0) {
    const int lane = threadIdx.x & 31;
    const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    CompressFlags fl;
    for (int64_t j0 = row0 + gw * 32; j0 < n; j0 += nw * 32) {
        const int64_t j = j0 + lane;
        bool long_row = false;
        if (j < n) {
            const int64_t s = ld(brm, j), e = ld(brm, j + 1);
            if (e - s > lane_max) {
                long_row = true;
            } else {
                int prev = INT_MIN, cw = -1, outn = 0;
                unsigned cm = 0;
                // entries in batches of 8 loaded ahead: the walk is bound by load latency
                // otherwise (ncu: 86 % long-scoreboard stalls)
                int cb8[8];
                for (int64_t q = s; q < e; ++q) {
                    if (((q - s) & 7) == 0) {
#pragma unroll
                        for (int u = 0; u < 8; ++u) cb8[u] = q + u < e ? __ldg(bent + q + u) : 0;
                    }
                    int col = cb8[0];
#pragma unroll
                    for (int u = 1; u < 8; ++u)
                        if (((q - s) & 7) == u) col = cb8[u];
                    fl.unsorted |= col < prev;
                    fl.nonstrict |= col <= prev;
                    fl.bad |= (col < 0) || ((int64_t)col >= k);
                    prev = col;
                    if (do_comp) {
                        const int w = col >> 5;
                        if (w != cw) {
                            if (cw >= 0) pairs[s + outn++] = make_uint2((unsigned)cw, cm);
                            cw = w;
                            cm = 0;
                        }
                        cm |= 1u << (col & 31);
                    }
                }
                if (do_comp) {
                    if (cw >= 0) pairs[s + outn++] = make_uint2((unsigned)cw, cm);
                    bc_len[j] = outn;
                    fl.words += (unsigned long long)outn;
                }
                if (bmeta) bmeta[j] = make_int4((int)(e - s), outn, s < e ? __ldg(bent + s) : INT_MAX, s < e ? prev : -1);
            }
        }
        unsigned lr = __ballot_sync(FULL, long_row);
        while (lr) {
            const int t = __ffs(lr) - 1;
            lr &= lr - 1;
            compress_row_warp(j0 + t, k, brm, bent, do_comp != 0, bc_len, pairs, bmeta, fl);
        }
    }
    if (__any_sync(FULL, fl.unsorted) && lane == 0) atomicAnd(&st->b_sorted, 0);
    if (__any_sync(FULL, fl.nonstrict) && lane == 0) atomicAnd(&st->b_strict, 0);
    if (validate && __any_sync(FULL, fl.bad) && lane == 0) atomicOr(&st->bad_index, 1);
    unsigned long long words = fl.words;
    for (int d = 16; d > 0; d >>= 1) words += __shfl_xor_sync(FULL, words, d);
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
                    int32_t* bc_len, uint2* pairs, int4* bmeta, DevStatus* st, int64_t row0) {
    if (B.nrows <= row0) return;
    const int threads = 256;
    const int grid = grid_for((B.nrows - row0 + 31) / 32, threads, L.num_sms, 16);
    // rows longer than lane_max are walked by the whole warp (coalesced, segmented OR scan);
    // shorter ones by one lane each (64 measured fastest on C2: 0.174 vs 0.250 ms at 32)
    const int lane_max = LANE_ROW_MAX;
    L.begin(do_comp ? "check_compress" : "check_sorted", L.stream);
    if (off64)
        k_check_compress<int64_t><<<grid, threads, 0, L.stream>>>(B.nrows, k, (const int64_t*)B.row_map, B.entries,
                                                                  do_comp, validate, bc_len, pairs, bmeta, st,
                                                                  lane_max, row0);
    else
        k_check_compress<int32_t><<<grid, threads, 0, L.stream>>>(B.nrows, k, (const int32_t*)B.row_map, B.entries,
                                                                  do_comp, validate, bc_len, pairs, bmeta, st,
                                                                  lane_max, row0);
    L.end(L.stream);
}

// ------------------------------------------------------------------------------------
// a1: per-row flops and the symbolic work bin of each row.
// A warp takes 32 consecutive rows of A, one per lane (long rows: the whole warp); per
// A entry one 16-byte gather of the B row's record (bmeta from a4; without it, the B
// row map).
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

// window bin for a row whose columns lie in [lo, hi] (sorted B), or 0: the smallest
// W in {8K, 16K, 32K, 48K, 64K, 128K, 192K} bits covering [lo & ~31, hi], used when clearing
// the window (W/32 words) costs at most ~16 words per bound insert and the row is not tiny.
__device__ __forceinline__ int sym_win_bin_of(int lo, int hi, int64_t ub) {
    if (hi < lo || ub <= 32) return 0;
    const int64_t span = (int64_t)hi - (int64_t)(lo & ~31) + 1;
    constexpr int64_t Ws[SYM_WIN_NBINS] = {8192, 16384, 32768, 49152, 65536, 131072, 196608};
    int c = 0;
    while (c < SYM_WIN_NBINS - 1 && Ws[c] < span) ++c;
    if (span > Ws[c] || Ws[c] / 32 > 16 * ub) return 0;
    return SYM_WIN_BIN0 + c;
}

struct FlopAcc {
    int64_t f = 0, fc = 0;
    int lo = INT_MAX, hi = -1;
    bool bad = false;
};

template <typename OffT>
__device__ __forceinline__ void flop_entry(int j, int64_t n, bool validate, const OffT* __restrict__ brm,
                                           const int32_t* __restrict__ bc_len, const int4* __restrict__ bmeta,
                                           bool comp, FlopAcc& acc) {
    if (validate && (j < 0 || (int64_t)j >= n)) {
        acc.bad = true;
        return;
    }
    if (bmeta) {
        const int4 m = __ldg(bmeta + j);
        acc.f += m.x;
        acc.fc += m.y;
        acc.lo = min(acc.lo, m.z);
        acc.hi = max(acc.hi, m.w);
    } else {
        acc.f += ld(brm, (int64_t)j + 1) - ld(brm, (int64_t)j);
        if (comp) acc.fc += __ldg(bc_len + j);
    }
}

template <typename OffT>
__global__ void __launch_bounds__(256) k_row_flops(int64_t m, int64_t n, int64_t k, const OffT* __restrict__ arm,
                                                   const int32_t* __restrict__ aent, const OffT* __restrict__ brm,
                                                   const int32_t* __restrict__ bc_len, int comp_mode, int64_t nnzB,
                                                   int validate, const int4* __restrict__ bmeta,
                                                   int64_t* __restrict__ flops, uint8_t* __restrict__ binid,
                                                   int32_t* __restrict__ counts, int32_t* __restrict__ wlo,
                                                   DevStatus* st, long long* __restrict__ pat_off) {
    bool comp = false;
    if (comp_mode == 1)
        comp = true;
    else if (comp_mode == -1)
        comp = nnzB > 0 && (st->total_words * 4ull <= (unsigned long long)nnzB * 3ull);
    // B_C rows are canonical (distinct increasing words) only for sorted B: the compressor
    // merges adjacent equal words, so an unsorted row can list a word twice, and the
    // symbolic kernels' plain read-OR-write rounds assume distinct words per B_C row.
    // Unsorted B therefore runs uncompressed (result-neutral).
    if (st->b_sorted == 0) comp = false;
    if (blockIdx.x == 0 && threadIdx.x == 0) st->use_comp = comp ? 1 : 0;
    const int lane = threadIdx.x & 31;
    const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int64_t kw = (k + 31) >> 5;
    const bool win = wlo != nullptr && bmeta != nullptr && st->b_sorted != 0;
    unsigned long long tot = 0;
    bool bad = false;
    for (int64_t i0 = gw * 32; i0 < m; i0 += nw * 32) {
        const int64_t i = i0 + lane;
        FlopAcc acc;
        bool long_row = false;
        if (i < m) {
            const int64_t s = ld(arm, i), e = ld(arm, i + 1);
            if (e - s > LANE_ROW_MAX) {
                long_row = true;
            } else {
                // 4 A entries (and their B-row records) in flight per lane: the walk is
                // bound by load latency otherwise (ncu: 72 % long-scoreboard stalls)
                int64_t p = s;
                for (; p + 4 <= e; p += 4) {
                    int jj[4];
#pragma unroll
                    for (int u = 0; u < 4; ++u) jj[u] = __ldg(aent + p + u);
#pragma unroll
                    for (int u = 0; u < 4; ++u) flop_entry(jj[u], n, validate, brm, bc_len, bmeta, comp, acc);
                }
                for (; p < e; ++p) flop_entry(__ldg(aent + p), n, validate, brm, bc_len, bmeta, comp, acc);
            }
        }
        unsigned lr = __ballot_sync(FULL, long_row);
        while (lr) {
            const int t = __ffs(lr) - 1;
            lr &= lr - 1;
            const int64_t it = i0 + t;
            const int64_t s = ld(arm, it), e = ld(arm, it + 1);
            FlopAcc w;
            for (int64_t p = s + lane; p < e; p += 32) flop_entry(__ldg(aent + p), n, validate, brm, bc_len, bmeta, comp, w);
            w.f = warp_sum(w.f);
            w.fc = warp_sum(w.fc);
            w.lo = __reduce_min_sync(FULL, w.lo);
            w.hi = __reduce_max_sync(FULL, w.hi);
            w.bad = __any_sync(FULL, w.bad);
            if (lane == t) acc = w;
        }
        if (i < m) {
            bad |= acc.bad;
            flops[i] = acc.f;
            const int64_t ub = comp ? min(acc.fc, kw) : min(acc.f, k);
            int b = sym_bin_of(ub);
            if (acc.f > 0 && acc.f <= TINY_MAX) {
                b = SYM_TINY_BIN;  // lane-owned register list (TinyList)
            } else if (win && b > 0) {
                const int wbn = sym_win_bin_of(acc.lo, acc.hi, ub);
                if (wbn) {
                    b = wbn;
                    wlo[i] = acc.lo & ~31;
                }
            }
            binid[i] = (uint8_t)b;
            if (pat_off) pat_off[i] = -1;  // no kept pattern yet (symbolic sets the kept ones)
            if (b == 0) counts[i] = 0;
            tot += (unsigned long long)acc.f;
        }
    }
    if (validate && __any_sync(FULL, bad) && lane == 0) atomicOr(&st->bad_index, 1);
    for (int d = 16; d > 0; d >>= 1) tot += __shfl_xor_sync(FULL, tot, d);
    if (lane == 0 && tot) atomicAdd(&st->total_flops, tot);
}

void row_flops_bin(Launch& L, bool off64, const MatView& A, const MatView& B, int64_t k, int comp_mode,
                   bool validate, const int32_t* bc_len, const int4* bmeta, int64_t* flops, uint8_t* binid,
                   int32_t* counts, int32_t* wlo, DevStatus* st, long long* pat_off) {
    if (A.nrows == 0) return;
    const int threads = 256;
    const int grid = grid_for((A.nrows + 31) / 32, threads, L.num_sms, 16);
    L.begin("row_flops_bin", L.stream);
    if (off64)
        k_row_flops<int64_t><<<grid, threads, 0, L.stream>>>(A.nrows, A.ncols, k, (const int64_t*)A.row_map,
                                                             A.entries, (const int64_t*)B.row_map, bc_len,
                                                             comp_mode, B.nnz, validate, bmeta, flops, binid, counts,
                                                             wlo, st, pat_off);
    else
        k_row_flops<int32_t><<<grid, threads, 0, L.stream>>>(A.nrows, A.ncols, k, (const int32_t*)A.row_map,
                                                             A.entries, (const int32_t*)B.row_map, bc_len,
                                                             comp_mode, B.nnz, validate, bmeta, flops, binid, counts,
                                                             wlo, st, pat_off);
    L.end(L.stream);
}

// ------------------------------------------------------------------------------------
// a2 / a6: exclusive scan in one pass (decoupled look-back), int64 accumulation.
// Tiles of SCAN_TILE items; a persistent grid of resident CTAs takes tiles in increasing
// order per CTA.  A tile publishes its aggregate, finds its exclusive prefix by walking back
// over its predecessors' published aggregates / inclusive prefixes, publishes its inclusive
// prefix and writes its outputs.  Flags carry a per-call epoch (no reset between calls).
// Deadlock-free because every tile below t is owned by a resident CTA that takes its tiles
// in increasing order (tile 0 never waits).
// ------------------------------------------------------------------------------------
constexpr int SCAN_THREADS = 512;
constexpr int SCAN_ITEMS = 8;
constexpr int SCAN_TILE = SCAN_THREADS * SCAN_ITEMS;

// per tile: flag (epoch << 2 | state), aggregate, inclusive prefix
int64_t scan_partial_len(int64_t m) { return 3 * ((m + SCAN_TILE - 1) / SCAN_TILE) + 4; }

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

constexpr long long SCAN_AGG = 1, SCAN_INCL = 2;

template <typename InT, typename OutT>
__global__ void __launch_bounds__(SCAN_THREADS) k_scan_lookback(int64_t m, const InT* __restrict__ in,
                                                                OutT* __restrict__ out, long long* __restrict__ tiles,
                                                                long long epoch, unsigned long long* total_dst,
                                                                int* overflow) {
    __shared__ long long s_prefix;
    const int64_t nb = (m + SCAN_TILE - 1) / SCAN_TILE;
    volatile long long* flag = tiles;  // tiles[3t], [3t+1] aggregate, [3t+2] inclusive prefix
    for (int64_t t = blockIdx.x; t < nb; t += gridDim.x) {
        const int64_t base = t * SCAN_TILE + (int64_t)threadIdx.x * SCAN_ITEMS;
        int64_t v[SCAN_ITEMS];
        int64_t sum = 0;
#pragma unroll
        for (int u = 0; u < SCAN_ITEMS; ++u) {
            const int64_t i = base + u;
            v[u] = i < m ? (int64_t)in[i] : 0;
            sum += v[u];
        }
        int64_t ex;
        const int64_t total = block_exclusive_scan(sum, &ex);
        if (threadIdx.x < 32) {
            // warp 0: publish the aggregate, then look back 32 predecessors at a time: wait
            // until all of the window are published, take the nearest inclusive prefix in it
            // (plus the aggregates after it), else all 32 aggregates and the next window
            const int lane = threadIdx.x;
            long long prefix = 0;
            if (lane == 0) {
                if (t == 0) {
                    tiles[2] = total;
                    __threadfence();
                    flag[0] = (epoch << 2) | SCAN_INCL;
                } else {
                    tiles[3 * t + 1] = total;
                    __threadfence();
                    flag[3 * t] = (epoch << 2) | SCAN_AGG;
                }
            }
            for (int64_t w = t - 1; w >= 0; w -= 32) {
                const int64_t p = w - lane;  // lane 0: the nearest predecessor
                long long f = 0;
                if (p >= 0) {
                    do {
                        f = flag[3 * p];
                    } while ((f >> 2) != epoch);
                }
                __threadfence();
                const unsigned incl = __ballot_sync(FULL, p >= 0 && (f & 3) == SCAN_INCL);
                const int stop = incl ? __ffs(incl) - 1 : 32;  // nearest lane holding an inclusive prefix
                long long v = 0;
                if (p >= 0 && lane < stop) v = ((volatile long long*)tiles)[3 * p + 1];
                if (p >= 0 && lane == stop) v = ((volatile long long*)tiles)[3 * p + 2];
                for (int d = 16; d > 0; d >>= 1) v += __shfl_xor_sync(FULL, v, d);
                prefix += v;
                if (incl) break;
            }
            if (lane == 0) {
                if (t > 0) {
                    tiles[3 * t + 2] = prefix + total;
                    __threadfence();
                    flag[3 * t] = (epoch << 2) | SCAN_INCL;
                }
                s_prefix = prefix;
            }
        }
        __syncthreads();
        int64_t run = s_prefix + ex;
#pragma unroll
        for (int u = 0; u < SCAN_ITEMS; ++u) {
            const int64_t i = base + u;
            if (i < m) out[i] = (OutT)run;
            run += v[u];
        }
        if (t == nb - 1 && threadIdx.x == 0) {
            const int64_t all = s_prefix + total;
            out[m] = (OutT)all;
            if (total_dst) *total_dst = (unsigned long long)all;
            if (sizeof(OutT) == 4 && all > (int64_t)INT_MAX && overflow) *overflow = 1;
        }
        __syncthreads();
    }
}

template <typename InT, typename OutT>
static void scan_t(Launch& L, const void* in, void* out, int64_t m, int64_t nb, long long* tiles, long long epoch,
                   unsigned long long* total_dst, int* overflow) {
    auto kern = k_scan_lookback<InT, OutT>;
    KCfg c = kernel_cfg(kern, SCAN_THREADS, 0, L.num_sms);
    const int grid = (int)std::min<int64_t>(nb, c.grid_cap);
    kern<<<grid, SCAN_THREADS, 0, L.stream>>>(m, (const InT*)in, (OutT*)out, tiles, epoch, total_dst, overflow);
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
    // a fresh epoch per call: flags left in the tile array by earlier calls never match; the
    // epochs start at a salted 60-bit value so that stale data in a reused buffer cannot
    // pass for a flag (flag = epoch << 2 | state)
    static std::atomic<long long> g_epoch{(long long)(0x0A5A5A5A5A000000ull ^
                                                      ((unsigned long long)(uintptr_t)&g_epoch << 12) ^
                                                      (unsigned long long)std::chrono::steady_clock::now()
                                                          .time_since_epoch()
                                                          .count()) &
                                          ((1ll << 60) - 1)};
    const long long epoch = g_epoch.fetch_add(1) & ((1ll << 60) - 1);
    long long* tiles = (long long*)partial;
    L.begin("exclusive_scan", L.stream);
    if (in64 && out64)
        scan_t<int64_t, int64_t>(L, in, out, m, nb, tiles, epoch, total_dst, overflow);
    else if (in64)
        scan_t<int64_t, int32_t>(L, in, out, m, nb, tiles, epoch, total_dst, overflow);
    else if (out64)
        scan_t<int32_t, int64_t>(L, in, out, m, nb, tiles, epoch, total_dst, overflow);
    else
        scan_t<int32_t, int32_t>(L, in, out, m, nb, tiles, epoch, total_dst, overflow);
    L.end(L.stream);
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
                                                       const long long* __restrict__ pat_off,
                                                       const int* __restrict__ pat_len, const uint2* __restrict__ pat,
                                                       const int64_t* __restrict__ flops,
                                                       uint8_t* __restrict__ binid, const DevStatus* st) {
    const bool use_pat = pat_off != nullptr && st->b_strict != 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
        int b = num_bin_of(counts[i]);
        if (b > 0 && flops && flops[i] <= TINY_MAX) {
            binid[i] = (uint8_t)NUM_TINY_BIN;
            continue;
        }
        if (use_pat && b >= 1 && b <= NUM_WARP_BINS) {
            const long long o = pat_off[i];
            if (o >= 0) {
                const int l = pat_len[i];
                const uint32_t span = l > 0 ? pat[o + l - 1].x - pat[o].x : 0u;
                b = span < (uint32_t)PAT_DENSE_WORDS ? NUM_PAT_BIN0 + b - 1 : NUM_PATH_BIN0 + max(b, 2) - 2;
            }
        }
        binid[i] = (uint8_t)b;
    }
}

void numeric_binid(Launch& L, int64_t m, const int32_t* counts, const long long* pat_off, const int* pat_len,
                   const uint2* pat, const int64_t* flops, uint8_t* binid, const DevStatus* st) {
    if (m == 0) return;
    int grid = (int)std::min<int64_t>((m + 255) / 256, (int64_t)L.num_sms * 16);
    L.begin("numeric_binid", L.stream);
    k_numeric_binid<<<grid, 256, 0, L.stream>>>(m, counts, pat_off, pat_len, pat, flops, binid, st);
    L.end(L.stream);
}

// Stable binning in tiles of BTILE rows (one CTA of BWARPS warps, BROWS rows per warp):
// pass 1 counts rows per bin per tile, pass 2 (one CTA) turns the counts into tile
// offsets per bin and the bin starts, pass 3 scatters rows in row order within a bin.
constexpr int BWARPS = 8;
constexpr int BROWS = 256;
constexpr int BTILE = BWARPS * BROWS;

int64_t bin_scratch_len(int64_t m) { return ((m + BTILE - 1) / BTILE) * NB + NB + 1; }

// per-warp histogram of its BROWS rows: lane b ends with the count of bin b
__device__ __forceinline__ int warp_bin_hist(int64_t r0, int64_t r1, const uint8_t* __restrict__ binid) {
    const int lane = threadIdx.x & 31;
    int cnt = 0;
    for (int64_t base = r0; base < r1; base += 32) {
        const int64_t r = base + lane;
        const int b = r < r1 ? (int)binid[r] : 255;
        // only the bins present among these 32 rows (usually one or two)
        unsigned pres = __reduce_or_sync(FULL, b < NB ? 1u << b : 0u);
        while (pres) {
            const int t = __ffs(pres) - 1;
            pres &= pres - 1;
            const unsigned bal = __ballot_sync(FULL, b == t);
            if (lane == t) cnt += __popc(bal);
        }
    }
    return cnt;
}

__global__ void __launch_bounds__(BWARPS * 32) k_bin_count(int64_t m, const uint8_t* __restrict__ binid,
                                                           int32_t* __restrict__ tilecnt) {
    __shared__ int wc[BWARPS][NB];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t r0 = (int64_t)blockIdx.x * BTILE + (int64_t)warp * BROWS, r1 = min(m, r0 + BROWS);
    const int cnt = r0 < m ? warp_bin_hist(r0, r1, binid) : 0;
    if (lane < NB) wc[warp][lane] = cnt;
    __syncthreads();
    if (threadIdx.x < NB) {
        int t = 0;
        for (int w = 0; w < BWARPS; ++w) t += wc[w][threadIdx.x];
        tilecnt[(int64_t)blockIdx.x * NB + threadIdx.x] = t;
    }
}

// one CTA, one warp per bin: exclusive scan of the bin's tile counts (all bins at once),
// then the bin starts from the bin totals
__global__ void __launch_bounds__(NB * 32) k_bin_offsets(int64_t ntiles, int32_t* __restrict__ tilecnt,
                                                         int* __restrict__ bin_start_dst) {
    __shared__ int64_t totals[NB];
    const int lane = threadIdx.x & 31, b = threadIdx.x >> 5;
    int64_t carry = 0;
    for (int64_t c0 = 0; c0 < ntiles; c0 += 32) {
        const int64_t c = c0 + lane;
        const int64_t v = c < ntiles ? tilecnt[c * NB + b] : 0;
        int64_t x = v;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const int64_t y = __shfl_up_sync(FULL, x, d);
            if (lane >= d) x += y;
        }
        if (c < ntiles) tilecnt[c * NB + b] = (int32_t)(carry + x - v);
        carry += __shfl_sync(FULL, x, 31);
    }
    if (lane == 0) totals[b] = carry;
    __syncthreads();
    if (threadIdx.x == 0) {
        int64_t run = 0;
        for (int t = 0; t < NB; ++t) {
            bin_start_dst[t] = (int)run;
            run += totals[t];
        }
        bin_start_dst[NB] = (int)run;
    }
}

__global__ void __launch_bounds__(BWARPS * 32) k_bin_scatter(int64_t m, const uint8_t* __restrict__ binid,
                                                             const int32_t* __restrict__ tilecnt,
                                                             const int* __restrict__ bin_start,
                                                             int32_t* __restrict__ perm) {
    __shared__ int wc[BWARPS][NB];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t r0 = (int64_t)blockIdx.x * BTILE + (int64_t)warp * BROWS, r1 = min(m, r0 + BROWS);
    const int cnt = r0 < m ? warp_bin_hist(r0, r1, binid) : 0;
    if (lane < NB) wc[warp][lane] = cnt;
    __syncthreads();
    int run = 0;
    if (lane < NB) {
        run = bin_start[lane] + tilecnt[(int64_t)blockIdx.x * NB + lane];
        for (int w = 0; w < warp; ++w) run += wc[w][lane];
    }
    for (int64_t base = r0; base < r1; base += 32) {
        const int64_t r = base + lane;
        const int b = r < r1 ? (int)binid[r] : 255;
        unsigned pres = __reduce_or_sync(FULL, b < NB ? 1u << b : 0u);
        while (pres) {
            const int t = __ffs(pres) - 1;
            pres &= pres - 1;
            const unsigned bal = __ballot_sync(FULL, b == t);
            const int base_t = __shfl_sync(FULL, run, t);
            if (b == t) perm[base_t + __popc(bal & lanemask_lt())] = (int32_t)r;
            if (lane == t) run += __popc(bal);
        }
    }
}

void bin_rows(Launch& L, int64_t m, const uint8_t* binid, int32_t* scratch, int32_t* perm, int* bin_start_dst) {
    const int64_t ntiles = (m + BTILE - 1) / BTILE;
    if (ntiles == 0) {
        cudaMemsetAsync(bin_start_dst, 0, sizeof(int) * (NB + 1), L.stream);
        return;
    }
    L.begin("bin_rows", L.stream);
    k_bin_count<<<(unsigned)ntiles, BWARPS * 32, 0, L.stream>>>(m, binid, scratch);
    k_bin_offsets<<<1, NB * 32, 0, L.stream>>>(ntiles, scratch, bin_start_dst);
    k_bin_scatter<<<(unsigned)ntiles, BWARPS * 32, 0, L.stream>>>(m, binid, scratch, bin_start_dst, perm);
    L.end(L.stream, 3);
}

// ------------------------------------------------------------------------------------
// Jacobi-fused numeric precondition ("all of its diagonal entries have
// nonzero values"): count rows of A without a stored A(i,i).  Validate mode only.
// ------------------------------------------------------------------------------------
template <typename OffT>
__global__ void __launch_bounds__(256) k_check_diag(int64_t m, const OffT* __restrict__ arm,
                                                    const int32_t* __restrict__ aent, int* __restrict__ missing) {
    const int lane = threadIdx.x & 31;
    const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    int miss = 0;
    for (int64_t i = gw; i < m; i += nw) {
        const int64_t s = ld(arm, i), e = ld(arm, i + 1);
        bool found = false;
        for (int64_t p = s + lane; p < e; p += 32) found |= __ldg(aent + p) == (int32_t)i;
        miss += __any_sync(FULL, found) ? 0 : 1;
    }
    if (lane == 0 && miss) atomicAdd(missing, miss);
}

bool check_diagonal(Launch& L, bool off64, int64_t m, const void* row_map, const int32_t* entries, int* scratch,
                    int* missing, int* missing_map) {
    *missing = 0;
    if (m == 0) return true;
    cudaMemsetAsync(scratch, 0, sizeof(int), L.stream);
    const int grid = (int)std::min<int64_t>((m * 32 + 255) / 256, (int64_t)L.num_sms * 8);
    L.begin("check_diag", L.stream);
    if (off64)
        k_check_diag<int64_t><<<grid, 256, 0, L.stream>>>(m, (const int64_t*)row_map, entries, scratch);
    else
        k_check_diag<int32_t><<<grid, 256, 0, L.stream>>>(m, (const int32_t*)row_map, entries, scratch);
    L.end(L.stream);
    const void* src = scratch;
    void* dst = missing_map;
    const size_t nb = sizeof(int);
    post_words(L, 1, &dst, &src, &nb);
    if (cudaStreamSynchronize(L.stream) != cudaSuccess) return false;
    *missing = *(volatile int*)missing;
    return true;
}

}  // namespace kk

// kk_num_hub.cu -- a7 + a8 for the dense bin (nnz(C_i) > 512) over a wide k: the paper's
// dense accumulator as a column bit vector in shared memory, and its
// two-level accumulator (level 1 in fast memory, level 2 for what does not
// fit) as (a) one CTA per row with the row's values in shared memory when they fit, and
// (b) a thread-block cluster per row for the rows that do not: the cluster's CTAs split the
// column range, exchange their slice counts through distributed shared memory, and
// accumulate their slices in their own shared memory (in rank windows when a slice is
// larger than one CTA's value array).  Global-memory atomics remain only as the fallback
// for unsorted B (no column-range search).
#include "kk_numeric.cuh"

#include <cooperative_groups.h>

#include <algorithm>
#include <cstdlib>

namespace kk {
namespace cg = cooperative_groups;

// ------------------------------------------------------------------------------------
// (a) k_num_hub: a CTA owns a row and the row's whole column bit vector (k bits) plus the
// popcount prefix of every group of 4 words in shared memory.  (1) the bit vector of the
// row's pattern (accum = OR, as the symbolic dense tier); (2) one pass over it writes the
// sorted column indices of C(i,:) and the group prefixes; (3) each product finds its rank
// in the row (group prefix + popcounts of <= 3 preceding words + the bits below it) and is
// added into the row's value array in shared memory (rows with nnz(C_i) <= vcap; fp64 add
// by compare-and-swap, 4 updates/clk/SM measured against 0.7 for L2 reductions), which is
// then written out coalesced.  Rows above vcap: skipped when the cluster tier takes them
// (big = 1), else added into C's values in global memory (fp64/fp32 reduction at L2).
// ------------------------------------------------------------------------------------
constexpr int HUB_THREADS = 1024;

// L2 residency hints for a long row's values accumulated at L2 (the zeroing stores and the
// reductions): evict_last keeps the row's value range in L2 while B's rows stream through,
// so the reductions do not re-read and re-write evicted lines in HBM
__device__ __forceinline__ unsigned long long l2_keep_policy() {
    unsigned long long p;
    asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ void red_add_keep(double* a, double v, unsigned long long pol) {
    asm volatile("red.global.add.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(a), "d"(v), "l"(pol) : "memory");
}
__device__ __forceinline__ void red_add_keep(float* a, float v, unsigned long long pol) {
    asm volatile("red.global.add.L2::cache_hint.f32 [%0], %1, %2;" ::"l"(a), "f"(v), "l"(pol) : "memory");
}
__device__ __forceinline__ void st_keep(double* a, double v, unsigned long long pol) {
    asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(a), "d"(v), "l"(pol) : "memory");
}
__device__ __forceinline__ void st_keep(float* a, float v, unsigned long long pol) {
    asm volatile("st.global.L2::cache_hint.f32 [%0], %1, %2;" ::"l"(a), "f"(v), "l"(pol) : "memory");
}
constexpr int HUB_WARPS = HUB_THREADS / 32;

// rank of column c in the row's bit vector: the prefix of its 4-word group plus the bits
// before it in the group (word loads as needed; one 16-byte load of the group measured
// slower on C4: num_hub 262 vs 253 ms)
__device__ __forceinline__ uint32_t hub_rank(const uint32_t* bm, const uint32_t* gp, int c) {
    const int w = c >> 5;
    uint32_t rk = gp[w >> 2];
    const int gw = w & ~3;
    if (gw + 0 < w) rk += __popc(bm[gw + 0]);
    if (gw + 1 < w) rk += __popc(bm[gw + 1]);
    if (gw + 2 < w) rk += __popc(bm[gw + 2]);
    return rk + __popc(bm[w] & ((1u << (c & 31)) - 1u));
}

__host__ __device__ constexpr int64_t hub_words(int64_t k) { return ((k + 127) / 128) * 4; }  // multiple of 4
constexpr int HUB_LONG = 256;  // B rows longer than this are walked by the whole CTA
constexpr int HUB_LIST = 1024; // capacity of the per-row list of such A entries
constexpr int HUB_HUGE = 1024; // listed B rows longer than this are walked by the whole CTA
constexpr int HUB_BATCH = 8;   // A entries per dynamically handed-out batch (short tails at the barrier)
constexpr int HUB_HLIST = 256; // capacity of the list of such rows (more: walked by one warp)

// shared layout: bm[NW] | gp[NW/4] (padded to 8 bytes) | wtot[HUB_WARPS] (int64) |
//                list[HUB_LIST] (int32) | nlist (+pad to 16) | hlist[HUB_HLIST] | vals[vcap]
__host__ __device__ constexpr int64_t hub_gp_words(int64_t k) { return (hub_words(k) / 4 + 1) & ~1ll; }
__host__ __device__ constexpr size_t hub_smem(int64_t k) {
    return (size_t)(hub_words(k) + hub_gp_words(k)) * 4 + (size_t)HUB_WARPS * 8 + (size_t)HUB_LIST * 4 + 16 +
           (size_t)HUB_HLIST * 4;
}

// The products of the A entries [s, e): each warp takes batches of 32 A entries (one
// load chain for the batch: column, value, B-row bounds per lane; batches handed out by a
// shared counter), then walks their B rows one after the other with 4 entries per lane in
// flight (otherwise the hub kernels are bound by load latency: one dependent chain per A
// entry per warp).  B rows longer than HUB_LONG are appended to the CTA's list and walked
// by all threads afterwards (a hub B row must not leave one warp working while the others
// wait at the barrier); when the list is full the warp walks the row itself.
// f(col, a * b) per product (b = 1 when VALS is false: the pattern pass loads no values).
template <int U, bool VALS, typename ValT, typename F>
__device__ __forceinline__ void hub_segment(const int32_t* __restrict__ bent, const ValT* __restrict__ bval,
                                            int64_t b0, int64_t len, int tid, int nthr, ValT a, F f) {
    for (int64_t x0 = tid; x0 < len; x0 += (int64_t)nthr * U) {
        int c[U];
        ValT v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t x = x0 + (int64_t)u * nthr;
            const bool ok = x < len;
            c[u] = ok ? __ldg(bent + b0 + x) : -1;
            v[u] = (VALS && ok) ? __ldg(bval + b0 + x) : (ValT)1;
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
            if (c[u] >= 0) f(c[u], a * v[u]);
    }
}

// nlist[0]: list length, nlist[1]: batch counter (both zero on entry).  ordered: the A
// entries one at a time by the whole CTA, in order, a barrier after each (deterministic mode:
// with strictly increasing B rows the products of one A entry have distinct columns, so
// f may add without atomics and every output sums its products in A order).
template <bool VALS, typename OffT, typename ValT, typename F>
__device__ __forceinline__ void hub_walk(int64_t s, int64_t e, const int32_t* __restrict__ aent,
                                         const ValT* __restrict__ aval, const OffT* __restrict__ brm,
                                         const int32_t* __restrict__ bent, const ValT* __restrict__ bval,
                                         int* list, int* nlist, F f, bool ordered = false) {
    const int lane = threadIdx.x & 31;
    if (ordered) {
        for (int64_t p = s; p < e; ++p) {
            const int j = __ldg(aent + p);
            const ValT a = VALS ? __ldg(aval + p) : (ValT)0;
            const int64_t bs = ld(brm, j), be = ld(brm, j + 1);
            hub_segment<4, VALS>(bent, bval, bs, be - bs, (int)threadIdx.x, HUB_THREADS, a, f);
            __syncthreads();
        }
        return;
    }
    while (true) {
        int b = 0;
        if (lane == 0) b = atomicAdd(nlist + 1, 1);
        const int64_t p0 = s + (int64_t)__shfl_sync(FULL, b, 0) * HUB_BATCH;
        if (p0 >= e) break;
        const int64_t p = p0 + lane;
        int64_t bs = 0, bl = 0;
        ValT a = (ValT)0;
        if (p < e && lane < HUB_BATCH) {
            const int j = __ldg(aent + p);
            if (VALS) a = __ldg(aval + p);
            bs = ld(brm, j);
            bl = ld(brm, j + 1) - bs;
        }
        // long B rows to the CTA list (one atomic per warp for the batch)
        const bool lng = bl > HUB_LONG;
        const unsigned lb = __ballot_sync(FULL, lng);
        bool listed = false;
        if (lb) {
            int base = 0;
            if (lane == 0) base = atomicAdd(nlist, __popc(lb));
            base = __shfl_sync(FULL, base, 0);
            const int slot = base + __popc(lb & lanemask_lt());
            if (lng && slot < HUB_LIST) {
                list[slot] = (int)(p - s);
                listed = true;
            }
        }
        const unsigned skip = __ballot_sync(FULL, listed);
        const int n = (int)min((int64_t)HUB_BATCH, e - p0);
        for (int t = 0; t < n; ++t) {
            if ((skip >> t) & 1u) continue;
            const int64_t tb = __shfl_sync(FULL, bs, t);
            const int64_t tl = __shfl_sync(FULL, bl, t);
            const ValT ta = __shfl_sync(FULL, a, t);
            hub_segment<8, VALS>(bent, bval, tb, tl, lane, 32, ta, f);
        }
    }
    __syncthreads();
    const int nl = min(*nlist, HUB_LIST);
    // listed rows of up to HUB_HUGE entries: one warp each, handed out by a counter (a CTA-wide
    // walk of a 300-entry row would leave most of the 1024 threads idle); longer ones are
    // re-listed at the front of the list and walked by the whole CTA
    while (true) {
        int l = 0;
        if (lane == 0) l = atomicAdd(nlist + 2, 1);
        l = __shfl_sync(FULL, l, 0);
        if (l >= nl) break;
        const int64_t p = s + list[l];
        const int j = __ldg(aent + p);
        const int64_t bs = ld(brm, j), be = ld(brm, j + 1);
        if (be - bs > HUB_HUGE) {
            int h = 0;
            if (lane == 0) h = atomicAdd(nlist + 3, 1);
            h = __shfl_sync(FULL, h, 0);
            if (h < HUB_HLIST) {
                if (lane == 0) nlist[4 + h] = (int)(p - s);
                continue;
            }
        }
        const ValT a = VALS ? __ldg(aval + p) : (ValT)0;
        hub_segment<8, VALS>(bent, bval, bs, be - bs, lane, 32, a, f);
    }
    __syncthreads();
    const int nh = min(nlist[3], HUB_HLIST);
    for (int l = 0; l < nh; ++l) {
        const int64_t p = s + nlist[4 + l];
        const int j = __ldg(aent + p);
        const ValT a = VALS ? __ldg(aval + p) : (ValT)0;
        const int64_t bs = ld(brm, j), be = ld(brm, j + 1);
        hub_segment<4, VALS>(bent, bval, bs, be - bs, (int)threadIdx.x, HUB_THREADS, a, f);
    }
}

template <typename OffT, typename ValT>
__global__ void __launch_bounds__(HUB_THREADS, 1) k_num_hub(const OffT* __restrict__ arm, const int32_t* __restrict__ aent,
                                                             const ValT* __restrict__ aval, const OffT* __restrict__ brm,
                                                             const int32_t* __restrict__ bent, const ValT* __restrict__ bval,
                                                             const OffT* __restrict__ crm, int32_t* __restrict__ cent,
                                                             ValT* __restrict__ cval, const int32_t* __restrict__ perm,
                                                             const int* __restrict__ bin_start, int bin, int64_t k,
                                                             int vcap, int big, int det,
                                                             const ValT* __restrict__ dinv, double omega,
                                                             int* __restrict__ row_ctr) {
    extern __shared__ __align__(16) uint32_t sm_hub[];
    const int64_t NW = hub_words(k);
    uint32_t* bm = sm_hub;
    uint32_t* gp = bm + NW;
    long long* wtot = (long long*)(gp + hub_gp_words(k));
    int* list = (int*)(wtot + HUB_WARPS);
    int* nlist = list + HUB_LIST;
    ValT* svals = (ValT*)(nlist + 4 + HUB_HLIST);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int r0 = bin_start[bin], r1 = bin_start[bin + 1];
    if (r0 + (int)blockIdx.x >= r1) return;
    const int64_t per = (NW / 4 + HUB_WARPS - 1) / HUB_WARPS * 4;  // words per warp (multiple of 4)
    const unsigned long long keep = l2_keep_policy();
    // rows handed out by a device counter (row_ctr) or round robin: they differ by two orders
    // of magnitude in work
    __shared__ int s_row;
    auto next_row = [&](int r) {
        if (!row_ctr) return r + (int)gridDim.x;
        __syncthreads();
        if (threadIdx.x == 0) s_row = r0 + (int)gridDim.x + atomicAdd(row_ctr, 1);
        __syncthreads();
        return s_row;
    };
    for (int r = r0 + blockIdx.x; r < r1;) {
        const int i = perm[r];
        const int64_t s = ld(arm, i), e = ld(arm, i + 1);
        const int64_t cb = ld(crm, i);
        const int64_t clen = ld(crm, i + 1) - cb;
        const bool inshared = clen <= (int64_t)vcap;
        if (!inshared && big) {  // the cluster tier's row
            r = next_row(r);
            continue;
        }
        for (int64_t t = threadIdx.x; t < NW / 4; t += HUB_THREADS) ((uint4*)bm)[t] = make_uint4(0, 0, 0, 0);
        if (threadIdx.x == 0) nlist[0] = nlist[1] = nlist[2] = nlist[3] = 0;
        __syncthreads();
        // (1) pattern (accum = OR)
        hub_walk<false>(s, e, aent, aval, brm, bent, bval, list, nlist,
                        [&](int c, ValT) { atomicOr(&bm[c >> 5], 1u << (c & 31)); });
        __syncthreads();
        // (2) per-warp ranges of 4-word groups: totals, then group prefixes + sorted entries in
        // one pass, a group per lane; chunks of 32 empty groups are skipped (their prefixes
        // are never read: no product falls in an empty group)
        const uint4* bm4 = (const uint4*)bm;
        const int64_t g0 = (int64_t)warp * (per / 4), g1 = min(NW / 4, g0 + per / 4);
        long long tot = 0;
        for (int64_t g = g0 + lane; g < g1; g += 32) {
            const uint4 v = bm4[g];
            tot += __popc(v.x) + __popc(v.y) + __popc(v.z) + __popc(v.w);
        }
        tot = warp_sum(tot);
        if (lane == 0) wtot[warp] = tot;
        __syncthreads();
        long long base = 0;
        for (int w = 0; w < warp; ++w) base += wtot[w];
        for (int64_t c0 = g0; c0 < g1; c0 += 32) {
            const int64_t g = c0 + lane;
            const uint4 v = g < g1 ? bm4[g] : make_uint4(0u, 0u, 0u, 0u);
            const int n = __popc(v.x) + __popc(v.y) + __popc(v.z) + __popc(v.w);
            if (__ballot_sync(FULL, n != 0) == 0u) continue;
            int x = n;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const int y = __shfl_up_sync(FULL, x, d);
                if (lane >= d) x += y;
            }
            long long pp = base + x - n;
            if (g < g1) gp[g] = (uint32_t)pp;
            const uint32_t wv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                uint32_t m = wv[u];
                while (m) {
                    const int b = __ffs(m) - 1;
                    m &= m - 1;
                    if (pp < clen) __stcs(cent + cb + pp, (int32_t)((g * 4 + u) * 32 + b));
                    ++pp;
                }
            }
            base += __shfl_sync(FULL, x, 31);
        }
        if (inshared)
            for (int64_t t = threadIdx.x; t < clen; t += HUB_THREADS) svals[t] = (ValT)0;
        else
            for (int64_t t = threadIdx.x; t < clen; t += HUB_THREADS) st_keep(cval + cb + t, (ValT)0, keep);
        if (threadIdx.x == 0) nlist[0] = nlist[1] = nlist[2] = nlist[3] = 0;
        __syncthreads();
        // (3) values: rank lookup, accumulation at the rank
        hub_walk<true>(s, e, aent, aval, brm, bent, bval, list, nlist, [&](int c, ValT prod) {
            const uint32_t rk = hub_rank(bm, gp, c);
            if ((int64_t)rk < clen) {
                if (det) {
                    if (inshared)
                        svals[rk] += prod;
                    else
                        cval[cb + rk] += prod;
                } else if (inshared) {
                    atomicAdd(&svals[rk], prod);
                } else {
                    red_add_keep(cval + cb + rk, prod, keep);
                }
            }
        }, det != 0);
        __syncthreads();
        if (dinv) {
            // Jacobi-fused row: C(i,:) = B(i,:) - omega D^-1(i) E(i,:): E(i,:)
            // scaled once by the row's scalar, then B(i,:) added at its ranks (its columns lie
            // in E's pattern when A(i,i) is stored; others are dropped)
            const ValT sc = (ValT)(-omega * (double)__ldg(dinv + i));
            if (inshared)
                for (int64_t t = threadIdx.x; t < clen; t += HUB_THREADS) svals[t] *= sc;
            else
                for (int64_t t = threadIdx.x; t < clen; t += HUB_THREADS) cval[cb + t] *= sc;
            __syncthreads();
            const int64_t bs = ld(brm, i), be = ld(brm, i + 1);
            for (int64_t q = bs + threadIdx.x; q < be; q += HUB_THREADS) {
                const int c = __ldg(bent + q);
                if (c < 0 || (int64_t)c >= k || !((bm[c >> 5] >> (c & 31)) & 1u)) continue;
                const uint32_t rk = hub_rank(bm, gp, c);
                if ((int64_t)rk >= clen) continue;
                const ValT b = __ldg(bval + q);
                if (det) {  // strictly increasing B(i,:): distinct ranks
                    if (inshared)
                        svals[rk] += b;
                    else
                        cval[cb + rk] += b;
                } else if (inshared) {
                    atomicAdd(&svals[rk], b);
                } else {
                    atomicAdd(&cval[cb + rk], b);
                }
            }
            __syncthreads();
        }
        if (inshared) {
            for (int64_t t = threadIdx.x; t < clen; t += HUB_THREADS) __stcs(cval + cb + t, svals[t]);
            __syncthreads();
        }
        r = next_row(r);
    }
}

// ------------------------------------------------------------------------------------
// (b) k_num_cluster: a cluster of CL_SIZE CTAs owns a row with nnz(C_i) > vcap of (a).
// CTA q of the cluster owns the column slice [q*S, (q+1)*S) of [0, k): its bit vector
// (S bits) and the group prefixes of the slice live in its shared memory.  Per row:
//   1. pattern: for every A entry, the B row's entries inside the slice (two warp-wide
//      searches in the sorted B row) set their bits (accum = OR);
//   2. the slice count goes to the CTA's shared memory, the cluster syncs, and each CTA
//      reads the counts of the CTAs before it through distributed shared memory (the
//      slice's offset in C(i,:)); the sorted column indices of the slice are written;
//   3. values: windows of vcap local ranks (most slices take one): per window, the B row
//      entries inside the window's column range are added at their rank into the CTA's
//      shared value array (fp64 add by compare-and-swap), which is written out coalesced.
// Rows are taken from a device counter by the cluster's CTA 0 and passed to the others
// through distributed shared memory (rows of the bin differ by two orders of magnitude in
// work).  Needs B's rows sorted (the column-range search).
// ------------------------------------------------------------------------------------
constexpr int CL_SIZE = 8;  // portable cluster size
constexpr int CL_THREADS = 512;
constexpr int CL_WARPS = CL_THREADS / 32;
constexpr int CL_LIST = 512;   // CTA-walked long B-row segments per pass
constexpr int CL_MAXWIN = 64;  // rank windows per slice

// columns per slice: a multiple of 256 (whole 4-word groups; the value array after the
// group prefixes stays 8-byte aligned)
__host__ __device__ constexpr int64_t cl_slice(int64_t k) { return ((k + CL_SIZE - 1) / CL_SIZE + 255) / 256 * 256; }

struct ClShared {
    int row[2];          // the cluster's current row (written by CTA 0, double-buffered)
    long long cnt[2];    // this CTA's slice count for the current row (double-buffered)
    long long off;       // offset of this CTA's slice in C(i,:)
    int nlist;
    int pad;
    long long wtot[CL_WARPS];
    int wcol[CL_MAXWIN + 1];  // first column of each rank window
    int2 list[CL_LIST];       // (lo - bs, hi - bs, A position) of long segments: .x lo, .y A offset
    int lhi[CL_LIST];
};

__host__ __device__ constexpr size_t cl_fixed_smem(int64_t k) {
    return (sizeof(ClShared) + 15) / 16 * 16 + (size_t)(cl_slice(k) / 32) * 4 + (size_t)(cl_slice(k) / 128) * 4;
}

// [lo, hi) of the entries of the sorted B row [bs, be) with columns in [c0, c1): warp-wide
// searches (32 probes per round)
__device__ __forceinline__ int64_t warp_lower_bound(const int32_t* __restrict__ bent, int64_t lo, int64_t hi, int64_t c) {
    const int lane = threadIdx.x & 31;
    while (hi - lo > 32) {
        const int64_t len = hi - lo;
        const int64_t pos = lo + (len * (lane + 1)) / 33;
        const unsigned b = __ballot_sync(FULL, (int64_t)__ldg(bent + pos) < c);
        const int n = __popc(b);
        const int64_t plo = __shfl_sync(FULL, pos, max(n - 1, 0));
        const int64_t phi = __shfl_sync(FULL, pos, min(n, 31));
        if (n > 0) lo = plo + 1;
        if (n < 32) hi = phi;
    }
    const int64_t q = lo + lane;
    const unsigned b = __ballot_sync(FULL, q < hi && (int64_t)__ldg(bent + q) < c);
    return lo + __popc(b);
}

__device__ __forceinline__ void warp_col_range(const int32_t* __restrict__ bent, int64_t bs, int64_t be, int64_t c0,
                                               int64_t c1, int64_t& lo, int64_t& hi) {
    const int lane = threadIdx.x & 31;
    if (be - bs <= 32) {
        const int64_t q = bs + lane;
        const int64_t c = q < be ? (int64_t)__ldg(bent + q) : INT64_MAX;
        lo = bs + __popc(__ballot_sync(FULL, c < c0));
        hi = bs + __popc(__ballot_sync(FULL, c < c1));
    } else {
        lo = warp_lower_bound(bent, bs, be, c0);
        hi = warp_lower_bound(bent, lo, be, c1);
    }
}

template <typename OffT, typename ValT>
__global__ void __launch_bounds__(CL_THREADS, 1)
    k_num_cluster(const OffT* __restrict__ arm, const int32_t* __restrict__ aent, const ValT* __restrict__ aval,
                  const OffT* __restrict__ brm, const int32_t* __restrict__ bent, const ValT* __restrict__ bval,
                  const OffT* __restrict__ crm, int32_t* __restrict__ cent, ValT* __restrict__ cval,
                  const int32_t* __restrict__ perm, const int* __restrict__ bin_start, int bin, int64_t k,
                  int64_t min_len, int vcap, int* __restrict__ row_ctr) {
    extern __shared__ __align__(16) unsigned char sm_cl[];
    cg::cluster_group cluster = cg::this_cluster();
    ClShared& S = *(ClShared*)sm_cl;
    const int64_t SL = cl_slice(k);
    const int SW = (int)(SL / 32);
    uint32_t* bm = (uint32_t*)(sm_cl + (sizeof(ClShared) + 15) / 16 * 16);
    uint32_t* gp = bm + SW;
    ValT* vals = (ValT*)(gp + SW / 4);
    const int q = (int)cluster.block_rank();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t cq0 = (int64_t)q * SL, cq1 = min(k, cq0 + SL);
    const int r0 = bin_start[bin], r1 = bin_start[bin + 1];
    const int per = (SW / 4 + CL_WARPS - 1) / CL_WARPS * 4;  // words per warp (multiple of 4)
    int parity = 0;
    while (true) {
        // the next row of the bin for the whole cluster
        if (q == 0 && threadIdx.x == 0) {
            int r;
            do {
                r = r0 + atomicAdd(row_ctr, 1);
            } while (r < r1 && ld(crm, perm[r] + 1) - ld(crm, perm[r]) <= min_len);
            S.row[parity] = r;
        }
        cluster.sync();
        const int r = *cluster.map_shared_rank(&S.row[parity], 0);
        if (r >= r1) break;
        const int i = perm[r];
        const int64_t s = ld(arm, i), e = ld(arm, i + 1);
        const int64_t cb = ld(crm, i);
        for (int t = threadIdx.x; t < SW / 4; t += CL_THREADS) ((uint4*)bm)[t] = make_uint4(0, 0, 0, 0);
        if (threadIdx.x == 0) S.nlist = 0;
        __syncthreads();
        // ---- 1. the slice's pattern bits ----
        auto set_bit = [&](int64_t c) {
            const int x = (int)(c - cq0);
            atomicOr(&bm[x >> 5], 1u << (x & 31));
        };
        for (int64_t p = s + warp; p < e; p += CL_WARPS) {
            const int j = __ldg(aent + p);
            const int64_t bs = ld(brm, j), be = ld(brm, j + 1);
            int64_t lo, hi;
            warp_col_range(bent, bs, be, cq0, cq1, lo, hi);
            if (hi - lo > HUB_LONG) {
                int slot = 0;
                if (lane == 0) slot = atomicAdd(&S.nlist, 1);
                slot = __shfl_sync(FULL, slot, 0);
                if (slot < CL_LIST) {
                    if (lane == 0) {
                        S.list[slot] = make_int2((int)(lo - bs), (int)(p - s));
                        S.lhi[slot] = (int)(hi - bs);
                    }
                    continue;
                }
            }
            for (int64_t x = lo + lane; x < hi; x += 32) set_bit(__ldg(bent + x));
        }
        __syncthreads();
        {
            const int nl = min(S.nlist, CL_LIST);
            for (int l = 0; l < nl; ++l) {
                const int j = __ldg(aent + s + S.list[l].y);
                const int64_t bs = ld(brm, j);
                for (int64_t x = bs + S.list[l].x + threadIdx.x; x < bs + S.lhi[l]; x += CL_THREADS)
                    set_bit(__ldg(bent + x));
            }
        }
        __syncthreads();
        // ---- 2. slice count, offset through distributed shared memory, columns ----
        const int w0 = warp * per, w1 = min(SW, w0 + per);
        long long tot = 0;
        for (int w = w0 + lane; w < w1; w += 32) tot += __popc(bm[w]);
        tot = warp_sum(tot);
        if (lane == 0) S.wtot[warp] = tot;
        __syncthreads();
        long long cnt = 0, base = 0;
        for (int w = 0; w < CL_WARPS; ++w) {
            if (w < warp) base += S.wtot[w];
            cnt += S.wtot[w];
        }
        if (threadIdx.x == 0) S.cnt[parity] = cnt;
        cluster.sync();
        if (threadIdx.x < 32) {
            long long o = 0;
            if (lane < q) o = *cluster.map_shared_rank(&S.cnt[parity], lane);
            o = warp_sum(o);
            if (lane == 0) S.off = o;
        }
        __syncthreads();
        const long long off = S.off;
        const int nwin = (int)((cnt + vcap - 1) / vcap);
        for (int c0 = w0; c0 < w1; c0 += 32) {
            const int w = c0 + lane;
            const uint32_t word = w < w1 ? bm[w] : 0u;
            const int n = __popc(word);
            int x = n;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const int y = __shfl_up_sync(FULL, x, d);
                if (lane >= d) x += y;
            }
            long long pos = base + x - n;
            if (w < w1 && (w & 3) == 0) gp[w >> 2] = (uint32_t)pos;
            uint32_t m = word;
            while (m) {
                const int b = __ffs(m) - 1;
                m &= m - 1;
                const int col = (int)(cq0 + (int64_t)w * 32 + b);
                __stcs(cent + cb + off + pos, (int32_t)col);
                if (pos % vcap == 0 && pos / vcap < CL_MAXWIN) S.wcol[pos / vcap] = col;
                ++pos;
            }
            base += __shfl_sync(FULL, x, 31);
        }
        if (threadIdx.x == 0) S.wcol[min(nwin, CL_MAXWIN)] = (int)cq1;
        __syncthreads();
        // ---- 3. values, window by window of vcap local ranks ----
        auto lrank = [&](int64_t c) -> int64_t {
            const int x = (int)(c - cq0);
            const int w = x >> 5;
            int64_t rk = gp[w >> 2];
            const int g0 = w & ~3;
            if (g0 + 0 < w) rk += __popc(bm[g0 + 0]);
            if (g0 + 1 < w) rk += __popc(bm[g0 + 1]);
            if (g0 + 2 < w) rk += __popc(bm[g0 + 2]);
            return rk + __popc(bm[w] & ((1u << (x & 31)) - 1u));
        };
        for (int win = 0; win < nwin; ++win) {
            const int64_t v0 = (int64_t)win * vcap;
            const int nv = (int)min((long long)vcap, cnt - v0);
            // window columns: ranks [v0, v0 + nv) <-> columns [wcol[win], wcol[win + 1])
            const int64_t wc0 = win < CL_MAXWIN ? S.wcol[win] : cq0;
            const int64_t wc1 = win + 1 < CL_MAXWIN ? S.wcol[min(win + 1, nwin)] : cq1;
            for (int t = threadIdx.x; t < nv; t += CL_THREADS) vals[t] = (ValT)0;
            if (threadIdx.x == 0) S.nlist = 0;
            __syncthreads();
            auto add = [&](int64_t c, ValT prod) {
                const int64_t lr = lrank(c) - v0;
                if (lr >= 0 && lr < nv) atomicAdd(&vals[lr], prod);
            };
            for (int64_t p = s + warp; p < e; p += CL_WARPS) {
                const int j = __ldg(aent + p);
                const int64_t bs = ld(brm, j), be = ld(brm, j + 1);
                int64_t lo, hi;
                warp_col_range(bent, bs, be, wc0, wc1, lo, hi);
                if (hi - lo > HUB_LONG) {
                    int slot = 0;
                    if (lane == 0) slot = atomicAdd(&S.nlist, 1);
                    slot = __shfl_sync(FULL, slot, 0);
                    if (slot < CL_LIST) {
                        if (lane == 0) {
                            S.list[slot] = make_int2((int)(lo - bs), (int)(p - s));
                            S.lhi[slot] = (int)(hi - bs);
                        }
                        continue;
                    }
                }
                const ValT a = __ldg(aval + p);
                for (int64_t x = lo + lane; x < hi; x += 32) add(__ldg(bent + x), a * __ldg(bval + x));
            }
            __syncthreads();
            {
                const int nl = min(S.nlist, CL_LIST);
                for (int l = 0; l < nl; ++l) {
                    const int64_t p = s + S.list[l].y;
                    const int j = __ldg(aent + p);
                    const ValT a = __ldg(aval + p);
                    const int64_t bs = ld(brm, j);
                    for (int64_t x = bs + S.list[l].x + threadIdx.x; x < bs + S.lhi[l]; x += CL_THREADS)
                        add(__ldg(bent + x), a * __ldg(bval + x));
                }
            }
            __syncthreads();
            for (int t = threadIdx.x; t < nv; t += CL_THREADS) __stcs(cval + cb + off + v0 + t, vals[t]);
            __syncthreads();
        }
        parity ^= 1;
    }
    // no CTA leaves while another may still read its shared memory
    cluster.sync();
}

// the cluster tier for rows above one CTA's value array: KK_HUB_CLUSTER=1 (measured slower
// than L2 reductions on C4; kept for the A/B and its parity test)
static bool use_cluster() {
    static const bool v = [] {
        const char* e = getenv("KK_HUB_CLUSTER");
        return e && e[0] == '1';
    }();
    return v;
}

template <typename OffT, typename ValT>
static bool hub_bins_t(Launch& L, const NumArgs& a, cudaStream_t s) {
    const size_t hsm = hub_smem(a.k);
    if (a.k <= 25600 || hsm > 200 * 1024) return false;
    const int drows = a.host_bin_start[NUM_DENSE_BIN + 1] - a.host_bin_start[NUM_DENSE_BIN];
    constexpr size_t SMEM_MAX = 227 * 1024;
    // (a) values of rows with nnz <= vcap in the CTA's shared memory
    int vcap = (int)std::min<size_t>((SMEM_MAX - hsm) / sizeof(ValT), (size_t)1 << 20);
    vcap = std::max(0, vcap - 64);
    const size_t hsm_v = hsm + (size_t)vcap * sizeof(ValT);
    // (b) the cluster tier for the longer rows: sorted B, slice bit vector + value window fit
    const size_t cfix = cl_fixed_smem(a.k);
    const int cvcap = cfix + 4096 * sizeof(ValT) <= SMEM_MAX ? (int)((SMEM_MAX - cfix) / sizeof(ValT)) - 64 : 0;
    const bool cluster = use_cluster() && !a.det && a.dinv == nullptr && a.sorted && a.work_ctr != nullptr && cvcap >= 4096;
    {
        auto kern = k_num_hub<OffT, ValT>;
        KCfg c = kernel_cfg(kern, HUB_THREADS, hsm_v, L.num_sms);
        const int grid = (int)std::min<int64_t>(drows, c.grid_cap);
        // rows from a device counter (C4: num_hub 270 -> 245 ms against round robin); the
        // cluster tier uses the counter itself
        int* rc = !cluster && a.work_ctr ? a.work_ctr : nullptr;
        if (rc) cudaMemsetAsync(rc, 0, sizeof(int), s);
        L.begin("num_hub", s);
        kern<<<grid, HUB_THREADS, hsm_v, s>>>((const OffT*)a.A.row_map, a.A.entries, (const ValT*)a.A.values,
                                              (const OffT*)a.B.row_map, a.B.entries, (const ValT*)a.B.values,
                                              (const OffT*)a.c_row_map, a.c_entries, (ValT*)a.c_values, a.perm,
                                              a.bin_start, NUM_DENSE_BIN, a.k, vcap, cluster ? 1 : 0,
                                              a.det ? 1 : 0, (const ValT*)a.dinv, a.omega, rc);
        L.end(s);
    }
    if (cluster) {
        const size_t csm = cfix + (size_t)cvcap * sizeof(ValT);
        auto kern = k_num_cluster<OffT, ValT>;
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)csm);
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(CL_SIZE, 1, 1);
        cfg.blockDim = dim3(CL_THREADS, 1, 1);
        cfg.dynamicSmemBytes = csm;
        cfg.stream = s;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = CL_SIZE;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        int nclusters = 0;
        if (cudaOccupancyMaxActiveClusters(&nclusters, (void*)kern, &cfg) != cudaSuccess || nclusters < 1) {
            cudaGetLastError();
            nclusters = std::max(1, L.num_sms / CL_SIZE);
        }
        nclusters = std::min(nclusters, drows);
        cfg.gridDim = dim3((unsigned)(nclusters * CL_SIZE), 1, 1);
        cudaMemsetAsync(a.work_ctr, 0, sizeof(int), s);
        L.begin(kname("num_cluster", nclusters), s);
        cudaLaunchKernelEx(&cfg, kern, (const OffT*)a.A.row_map, a.A.entries, (const ValT*)a.A.values,
                           (const OffT*)a.B.row_map, a.B.entries, (const ValT*)a.B.values, (const OffT*)a.c_row_map,
                           a.c_entries, (ValT*)a.c_values, a.perm, a.bin_start, (int)NUM_DENSE_BIN, a.k,
                           (int64_t)vcap, cvcap, a.work_ctr);
        L.end(s);
    }
    return true;
}

bool launch_hub_bins(Launch& L, const NumArgs& a, cudaStream_t s) {
    if (a.off64) {
        if (a.f64) return hub_bins_t<int64_t, double>(L, a, s);
        return hub_bins_t<int64_t, float>(L, a, s);
    }
    if (a.f64) return hub_bins_t<int32_t, double>(L, a, s);
    return hub_bins_t<int32_t, float>(L, a, s);
}

}  // namespace kk

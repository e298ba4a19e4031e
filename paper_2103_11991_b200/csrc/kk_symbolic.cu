// kk_symbolic.cu -- a5: symbolic phase (bit vector PAPER.md:180).
//
//   k_sym_warp<S>   warp-owned shared-memory hash over B_C words, accum = OR
//   k_sym_dense     CTA-owned dense bit vector over column windows
#include "kk_device.cuh"

#include <type_traits>

namespace kk {
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

// a5 for rows whose bound exceeds the warp tables: the paper's dense bit-vector
// accumulator in one CTA's shared memory, over windows of `wbits`
// columns when k is larger.  Sorted B rows are resumed from per-entry cursors.
template <typename OffT>
__global__ void __launch_bounds__(1024) k_sym_dense(const OffT* __restrict__ arm, const int32_t* __restrict__ aent,
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
    // single-window rows: A entries whose B(_C) row is long are listed and walked by the
    // whole CTA afterwards, so one hub B row does not hold the other warps at the barrier
    constexpr int LONG = 256, LIST = 1024;
    int* list = (int*)(bmp + maxw);
    int* nlist = list + LIST;
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
            if (threadIdx.x == 0) *nlist = 0;
            __syncthreads();
            if (single) {
                // one window over all of k: batches of 32 A entries per warp (one load chain per
                // batch), their B(_C) rows walked with 8 entries per lane in flight; long rows to
                // the CTA list (the walk is bound by load latency otherwise)
                for (int64_t p0 = s + (int64_t)warp * 32; p0 < e; p0 += (int64_t)warps * 32) {
                    const int64_t p = p0 + lane;
                    int64_t bs = 0, len = 0;
                    if (p < e) {
                        const int j = __ldg(aent + p);
                        bs = ld(brm, j);
                        len = comp ? __ldg(bc_len + j) : ld(brm, j + 1) - bs;
                    }
                    const bool lng = len > LONG;
                    const unsigned lb = __ballot_sync(FULL, lng);
                    bool listed = false;
                    if (lb) {
                        int base = 0;
                        if (lane == 0) base = atomicAdd(nlist, __popc(lb));
                        base = __shfl_sync(FULL, base, 0);
                        const int slot = base + __popc(lb & lanemask_lt());
                        if (lng && slot < LIST) {
                            list[slot] = (int)(p - s);
                            listed = true;
                        }
                    }
                    const unsigned skip = __ballot_sync(FULL, listed);
                    const int n = (int)min((int64_t)32, e - p0);
                    for (int t = 0; t < n; ++t) {
                        if ((skip >> t) & 1u) continue;
                        const int64_t tb = __shfl_sync(FULL, bs, t);
                        const int64_t tl = __shfl_sync(FULL, len, t);
                        for (int64_t x0 = lane; x0 < tl; x0 += 32 * 8) {
                            if (comp) {
                                uint2 pr[8];
#pragma unroll
                                for (int u = 0; u < 8; ++u)
                                    pr[u] = x0 + 32 * u < tl ? __ldg(pairs + tb + x0 + 32 * u) : make_uint2(0u, 0u);
#pragma unroll
                                for (int u = 0; u < 8; ++u)
                                    if (pr[u].y) atomicOr(&bmp[pr[u].x], pr[u].y);
                            } else {
                                int c[8];
#pragma unroll
                                for (int u = 0; u < 8; ++u) c[u] = x0 + 32 * u < tl ? __ldg(bent + tb + x0 + 32 * u) : -1;
#pragma unroll
                                for (int u = 0; u < 8; ++u)
                                    if (c[u] >= 0) atomicOr(&bmp[c[u] >> 5], 1u << (c[u] & 31));
                            }
                        }
                    }
                }
            }
            for (int64_t p = s + warp; p < e && !single; p += warps) {
                const int j = __ldg(aent + p);
                const int64_t bs = ld(brm, j);
                if (single) {
                    const int64_t len = comp ? __ldg(bc_len + j) : ld(brm, j + 1) - bs;
                    if (len > LONG) {
                        int slot = 0;
                        if (lane == 0) slot = atomicAdd(nlist, 1);
                        slot = __shfl_sync(FULL, slot, 0);
                        if (slot < LIST) {
                            if (lane == 0) list[slot] = (int)(p - s);
                            continue;
                        }
                    }
                }
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
            if (single) {
                const int nl = min(*nlist, LIST);
                for (int l = 0; l < nl; ++l) {
                    const int j = __ldg(aent + s + list[l]);
                    const int64_t bs = ld(brm, j);
                    if (comp) {
                        const int64_t be = bs + __ldg(bc_len + j);
                        for (int64_t q = bs + threadIdx.x; q < be; q += blockDim.x) {
                            const uint2 pr = __ldg(pairs + q);
                            atomicOr(&bmp[pr.x], pr.y);
                        }
                    } else {
                        const int64_t be = ld(brm, j + 1);
                        for (int64_t q = bs + threadIdx.x; q < be; q += blockDim.x) {
                            const int c = __ldg(bent + q);
                            atomicOr(&bmp[c >> 5], 1u << (c & 31));
                        }
                    }
                }
                __syncthreads();
            }
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

static int sym_warps_for(int S) { return S <= 512 ? 8 : (S == 1024 ? 4 : (S == 2048 ? 2 : 1)); }

// rows of symbolic bin `bin` when the host holds the bin starts (else -1: launch anyway)
static inline int64_t host_rows(const SymArgs& a, int bin) {
    return a.host_bin_start ? (int64_t)a.host_bin_start[bin + 1] - a.host_bin_start[bin] : -1;
}

template <typename OffT, int S>
static void launch_sym_warp(Launch& L, const SymArgs& a, int bin) {
    const int warps = sym_warps_for(S);
    const size_t smem = (size_t)warps * 2 * S * sizeof(uint32_t);
    auto kern = k_sym_warp<OffT, S>;
    KCfg c = kernel_cfg(kern, warps * 32, smem, L.num_sms);
    int grid = c.grid_cap;
    const int64_t hr = host_rows(a, bin);
    if (hr == 0) return;
    int64_t need = ((hr > 0 ? hr : a.A.nrows) + warps - 1) / warps;
    if (need < grid) grid = (int)(need > 0 ? need : 1);
    L.begin(kname("sym_warp", S), L.stream);
    kern<<<grid, warps * 32, smem, L.stream>>>((const OffT*)a.A.row_map, a.A.entries, (const OffT*)a.B.row_map,
                                               a.B.entries, a.bc_len, a.pairs, a.perm, a.bin_start, bin, a.logG,
                                               a.counts, a.st);
    L.end(L.stream);
}


// ------------------------------------------------------------------------------------
// a5 for rows of sorted B whose columns fit a window of W bits: the paper's dense bit
// vector, one per warp, over [wlo, wlo + W).  One B_C row per step: its
// words are distinct (B_C of a sorted row is canonical), so each lane ORs its mask with
// a plain shared load/store and counts the bits it adds (popc(mask & ~old)).  Without
// compression the lanes of a step can share a word, so the OR is atomic instead.
// Words that turn non-zero are appended to a per-warp list; at the end of the row the
// list (<= PL words) is sorted and the row's pattern -- its (word, mask) pairs in column
// order -- is kept in the handle for the numeric phase (symbolic state carried by the
// handle), and only the listed words are cleared.  Rows with more
// than PL words clear the whole window and keep no pattern.
// ------------------------------------------------------------------------------------
constexpr int PAT_WORDS = 64;  // max words of a stored row pattern
constexpr int FLAT_WORDS = 512;  // room for the flattened pair offsets of a chunk

// Per A entry of the chunk: start (element offset into B_C pairs or B entries) and length
// of its B row; O32 when offsets fit 31 bits (cheaper 32-bit addressing).
template <bool O32>
struct SymRec;
template <>
struct __align__(8) SymRec<true> {
    int bb;
    int len;
};
template <>
struct __align__(16) SymRec<false> {
    long long bb;
    int len;
    int pad;
};

template <typename OffT, int W, bool COMP, bool O32>
__device__ __forceinline__ void sym_window_rows(const OffT* __restrict__ arm, const int32_t* __restrict__ aent,
                                                const OffT* __restrict__ brm, const int32_t* __restrict__ bent,
                                                const int32_t* __restrict__ bc_len, const uint2* __restrict__ pairs,
                                                const int32_t* __restrict__ perm, int r0, int r1,
                                                const int32_t* __restrict__ wlo, int32_t* __restrict__ counts,
                                                uint32_t* bm, void* rec_raw, uint32_t* wl, const PatOut& po,
                                                DevStatus* st) {
    using SR = SymRec<O32>;
    SR* rec = (SR*)rec_raw;
    // flattened pair offsets of a chunk (FLAT_CAP entries of SR::bb), per-lane scratch
    decltype(SR::bb)* flat = (decltype(SR::bb)*)((uint32_t*)rec_raw + 128);
    uint32_t* scratch = (uint32_t*)rec_raw + 128 + FLAT_WORDS;
    constexpr int NW = W / 32;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, warps = blockDim.x >> 5;
    const int stride = gridDim.x * warps;
    int r = r0 + blockIdx.x * warps + warp;
    // software pipeline over rows: the next row's bounds and first 32 A entries are
    // loaded while the current row finishes
    int i = perm[r];
    int64_t s = ld(arm, i), e = ld(arm, i + 1);
    int jn = lane < e - s ? __ldg(aent + s + lane) : 0;
    while (true) {
        const uint32_t wb = (uint32_t)__ldg(wlo + i) >> 5;
        const int rn = r + stride;
        const int inext = rn < r1 ? perm[rn] : -1;
        int cnt = 0;
        int nt = 0;  // words touched (warp-uniform)
        auto step_or = [&](uint32_t w, uint32_t m) {
            bool fresh = false;
            uint32_t x = 0;
            if (m) {
                x = w - wb;
                uint32_t old;
                if (COMP) {
                    old = bm[x];
                    bm[x] = old | m;
                } else {
                    old = atomicOr(&bm[x], m);
                }
                cnt += __popc(m & ~old);
                fresh = old == 0;
            }
            const unsigned fb = __ballot_sync(FULL, fresh);
            if (fresh) {
                const int pos = nt + __popc(fb & lanemask_lt());
                if (pos < PAT_WORDS) wl[pos] = x;
            }
            nt += __popc(fb);
        };
        for (int64_t c0 = s; c0 < e; c0 += 32) {
            const int na = (int)min((int64_t)32, e - c0);
            int j = jn;
            if (c0 != s && lane < na) j = __ldg(aent + c0 + lane);
            int bl = 0;
            __syncwarp();
            if (lane < na) {
                const int64_t bb = ld(brm, j);
                bl = COMP ? __ldg(bc_len + j) : (int)(ld(brm, j + 1) - bb);
                SR sr;
                sr.bb = (decltype(sr.bb))bb;
                sr.len = bl;
                rec[lane] = sr;
            }
            const int maxbl = (int)__reduce_max_sync(FULL, (unsigned)bl);
            __syncwarp();
            if (maxbl == 0) continue;
            auto load = [&](const SR& sr, int q, uint32_t& w, uint32_t& m) {
                if (COMP) {
                    const uint2 pr = __ldg(pairs + (sr.bb + q));
                    w = pr.x;
                    m = pr.y;
                } else {
                    const int c = __ldg(bent + (sr.bb + q));
                    w = (uint32_t)c >> 5;
                    m = 1u << (c & 31);
                }
            };
            // pairs of the chunk's B_C rows, flattened: 32 consecutive pairs per step
            int incl = bl;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const int y = __shfl_up_sync(FULL, incl, d);
                if (lane >= d) incl += y;
            }
            const int U = __shfl_sync(FULL, incl, 31);
            constexpr int FLAT_CAP = FLAT_WORDS * 4 / (int)sizeof(SR::bb);  // else one B row per step
            if (U <= FLAT_CAP) {
                if (lane < na) {
                    const SR sr = rec[lane];
                    for (int q = 0, ex = incl - bl; q < bl; ++q) flat[ex + q] = sr.bb + q;
                }
                __syncwarp();
                int u0 = 0;
                auto fetch = [&](uint32_t& w, uint32_t& m) {
                    w = 0;
                    m = 0;
                    if (u0 >= U) return false;
                    const int p = u0 + lane;
                    u0 += 32;
                    if (p < U) {
                        SR one;
                        one.bb = flat[p];
                        load(one, 0, w, m);
                    }
                    return true;
                };
                // equal words in a step are merged (match + OR over the group); the group
                // leader updates the bit vector, so all updates of a step are distinct words
                auto step_merge = [&](uint32_t w, uint32_t m) {
                    const uint32_t x = w - wb;
                    const uint32_t key = m ? x : (0x80000000u | (uint32_t)lane);
                    const unsigned grp = __match_any_sync(FULL, key);
                    scratch[lane] = m;
                    __syncwarp();
                    uint32_t mm = m;
                    bool fresh = false;
                    if (m && lane == __ffs(grp) - 1) {
                        unsigned peers = grp & (grp - 1);  // the group without its leader
                        while (peers) {
                            mm |= scratch[__ffs(peers) - 1];
                            peers &= peers - 1;
                        }
                        const uint32_t old = bm[x];
                        bm[x] = old | mm;
                        cnt += __popc(mm & ~old);
                        fresh = old == 0;
                    }
                    const unsigned fb = __ballot_sync(FULL, fresh);
                    if (fresh) {
                        const int pos = nt + __popc(fb & lanemask_lt());
                        if (pos < PAT_WORDS) wl[pos] = x;
                    }
                    nt += __popc(fb);
                };
                uint32_t w0, w1, w2, w3, m0, m1, m2, m3;
                fetch(w0, m0);
                bool h1 = fetch(w1, m1);
                bool h2 = fetch(w2, m2);
                bool h3 = fetch(w3, m3);
                while (true) {
                    step_merge(w0, m0);
                    if (!h1) break;
                    __syncwarp();
                    const bool h0 = fetch(w0, m0);
                    step_merge(w1, m1);
                    if (!h2) break;
                    __syncwarp();
                    h1 = fetch(w1, m1);
                    step_merge(w2, m2);
                    if (!h3) break;
                    __syncwarp();
                    h2 = fetch(w2, m2);
                    step_merge(w3, m3);
                    if (!h0) break;
                    __syncwarp();
                    h3 = fetch(w3, m3);
                }
            } else {
                for (int t = 0; t < na; ++t) {
                    const SR sr = rec[t];
                    for (int q0 = 0; q0 < sr.len; q0 += 32) {
                        uint32_t w = 0, m = 0;
                        if (q0 + lane < sr.len) load(sr, q0 + lane, w, m);
                        step_or(w, m);
                        __syncwarp();
                    }
                }
            }
            __syncwarp();
        }
        int64_t sn = 0, en = 0;
        if (inext >= 0) {
            sn = ld(arm, inext);
            en = ld(arm, inext + 1);
        }
        cnt = warp_sum(cnt);
        if (lane == 0) counts[i] = cnt;
        __syncwarp();
        if (nt <= PAT_WORDS) {
            // sort the touched words (relative indices < NW), store the pattern, clear them
            constexpr int E = PAT_WORDS / 32;
            uint32_t v[E];
#pragma unroll
            for (int q = 0; q < E; ++q) {
                const int idx = lane * E + q;
                v[q] = idx < nt ? wl[idx] : 0xffffffffu;
            }
            warp_bitonic_sort<E>(v);
            long long off = -1;
            if (po.pat) {
                if (lane == 0) {
                    const unsigned long long o = atomicAdd(&st->pat_used, (unsigned long long)nt);
                    off = (o + (unsigned long long)nt <= (unsigned long long)po.cap) ? (long long)o : -1;
                }
                off = __shfl_sync(FULL, off, 0);
            }
#pragma unroll
            for (int q = 0; q < E; ++q) {
                const int idx = lane * E + q;
                if (idx < nt) {
                    const uint32_t x = v[q];
                    const uint32_t m = bm[x];
                    bm[x] = 0;
                    if (off >= 0) po.pat[off + idx] = make_uint2(x + wb, m);
                }
            }
            if (po.pat && lane == 0) {
                po.off[i] = off;
                po.len[i] = nt;
            }
        } else {
            for (int t = lane; t < NW / 4; t += 32) ((uint4*)bm)[t] = make_uint4(0, 0, 0, 0);
        }
        if (inext >= 0) jn = lane < en - sn ? __ldg(aent + sn + lane) : 0;
        __syncwarp();
        if (inext < 0) break;
        r = rn;
        i = inext;
        s = sn;
        e = en;
    }
}

// a5 on a warp-owned hash table of B_C words (keys[S] | masks[S]) -- the structure of
// sym_window_rows (flattened pairs, match-merged duplicate words, touched-word list,
// kept patterns) for rows whose columns do not fit a bit-vector window.  Leaders claim
// new words with write-then-verify (strict_claim); the list holds slots.
template <typename OffT, int S, bool COMP, bool O32>
__device__ __forceinline__ void sym_hash_rows(const OffT* __restrict__ arm, const int32_t* __restrict__ aent,
                                                const OffT* __restrict__ brm, const int32_t* __restrict__ bent,
                                                const int32_t* __restrict__ bc_len, const uint2* __restrict__ pairs,
                                                const int32_t* __restrict__ perm, int r0, int r1,
                                                int32_t* __restrict__ counts,
                                                uint32_t* keys, uint32_t* masks, void* rec_raw, uint32_t* wl,
                                                const PatOut& po, DevStatus* st) {
    using SR = SymRec<O32>;
    SR* rec = (SR*)rec_raw;
    // flattened pair offsets of a chunk (FLAT_CAP entries of SR::bb), per-lane scratch
    decltype(SR::bb)* flat = (decltype(SR::bb)*)((uint32_t*)rec_raw + 128);
    uint32_t* scratch = (uint32_t*)rec_raw + 128 + FLAT_WORDS;
    constexpr int LOGS = ilog2(S);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, warps = blockDim.x >> 5;
    const int stride = gridDim.x * warps;
    int r = r0 + blockIdx.x * warps + warp;
    // software pipeline over rows: the next row's bounds and first 32 A entries are
    // loaded while the current row finishes
    int i = perm[r];
    int64_t s = ld(arm, i), e = ld(arm, i + 1);
    int jn = lane < e - s ? __ldg(aent + s + lane) : 0;
    while (true) {
        const int rn = r + stride;
        const int inext = rn < r1 ? perm[rn] : -1;
        int cnt = 0;
        int nt = 0;  // words touched (warp-uniform)
        auto step_or = [&](uint32_t w, uint32_t m) {
            // one B row segment: words distinct (COMP); raw columns may repeat a word, so
            // they are merged first exactly like the flattened path
            const uint32_t key = m ? w : (0x80000000u | (uint32_t)lane);
            const unsigned grp = COMP ? (1u << lane) : __match_any_sync(FULL, key);
            scratch[lane] = m;
            __syncwarp();
            uint32_t mm = m;
            const bool lead = m && lane == __ffs(grp) - 1;
            if (lead) {
                unsigned peers = grp & (grp - 1);
                while (peers) {
                    mm |= scratch[__ffs(peers) - 1];
                    peers &= peers - 1;
                }
            }
            const uint32_t hs = strict_claim<S>(keys, w, lead);
            bool fresh = false;
            if (lead) {
                const uint32_t old = masks[hs];
                masks[hs] = old | mm;
                cnt += __popc(mm & ~old);
                fresh = old == 0;
            }
            const unsigned fb = __ballot_sync(FULL, fresh);
            if (fresh) {
                const int pos = nt + __popc(fb & lanemask_lt());
                if (pos < PAT_WORDS) wl[pos] = hs;
            }
            nt += __popc(fb);
        };
        for (int64_t c0 = s; c0 < e; c0 += 32) {
            const int na = (int)min((int64_t)32, e - c0);
            int j = jn;
            if (c0 != s && lane < na) j = __ldg(aent + c0 + lane);
            int bl = 0;
            __syncwarp();
            if (lane < na) {
                const int64_t bb = ld(brm, j);
                bl = COMP ? __ldg(bc_len + j) : (int)(ld(brm, j + 1) - bb);
                SR sr;
                sr.bb = (decltype(sr.bb))bb;
                sr.len = bl;
                rec[lane] = sr;
            }
            const int maxbl = (int)__reduce_max_sync(FULL, (unsigned)bl);
            __syncwarp();
            if (maxbl == 0) continue;
            auto load = [&](const SR& sr, int q, uint32_t& w, uint32_t& m) {
                if (COMP) {
                    const uint2 pr = __ldg(pairs + (sr.bb + q));
                    w = pr.x;
                    m = pr.y;
                } else {
                    const int c = __ldg(bent + (sr.bb + q));
                    w = (uint32_t)c >> 5;
                    m = 1u << (c & 31);
                }
            };
            // pairs of the chunk's B_C rows, flattened: 32 consecutive pairs per step
            int incl = bl;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const int y = __shfl_up_sync(FULL, incl, d);
                if (lane >= d) incl += y;
            }
            const int U = __shfl_sync(FULL, incl, 31);
            constexpr int FLAT_CAP = FLAT_WORDS * 4 / (int)sizeof(SR::bb);  // else one B row per step
            if (U <= FLAT_CAP) {
                if (lane < na) {
                    const SR sr = rec[lane];
                    for (int q = 0, ex = incl - bl; q < bl; ++q) flat[ex + q] = sr.bb + q;
                }
                __syncwarp();
                int u0 = 0;
                auto fetch = [&](uint32_t& w, uint32_t& m) {
                    w = 0;
                    m = 0;
                    if (u0 >= U) return false;
                    const int p = u0 + lane;
                    u0 += 32;
                    if (p < U) {
                        SR one;
                        one.bb = flat[p];
                        load(one, 0, w, m);
                    }
                    return true;
                };
                // equal words in a step are merged (match + OR over the group); the group
                // leader updates the bit vector, so all updates of a step are distinct words
                auto step_merge = [&](uint32_t w, uint32_t m) {
                    const uint32_t key = m ? w : (0x80000000u | (uint32_t)lane);
                    const unsigned grp = __match_any_sync(FULL, key);
                    scratch[lane] = m;
                    __syncwarp();
                    uint32_t mm = m;
                    const bool lead = m && lane == __ffs(grp) - 1;
                    if (lead) {
                        unsigned peers = grp & (grp - 1);
                        while (peers) {
                            mm |= scratch[__ffs(peers) - 1];
                            peers &= peers - 1;
                        }
                    }
                    const uint32_t hs = strict_claim<S>(keys, w, lead);
                    bool fresh = false;
                    if (lead) {
                        const uint32_t old = masks[hs];
                        masks[hs] = old | mm;
                        cnt += __popc(mm & ~old);
                        fresh = old == 0;
                    }
                    const unsigned fb = __ballot_sync(FULL, fresh);
                    if (fresh) {
                        const int pos = nt + __popc(fb & lanemask_lt());
                        if (pos < PAT_WORDS) wl[pos] = hs;
                    }
                    nt += __popc(fb);
                };
                uint32_t w0, w1, w2, w3, m0, m1, m2, m3;
                fetch(w0, m0);
                bool h1 = fetch(w1, m1);
                bool h2 = fetch(w2, m2);
                bool h3 = fetch(w3, m3);
                while (true) {
                    step_merge(w0, m0);
                    if (!h1) break;
                    __syncwarp();
                    const bool h0 = fetch(w0, m0);
                    step_merge(w1, m1);
                    if (!h2) break;
                    __syncwarp();
                    h1 = fetch(w1, m1);
                    step_merge(w2, m2);
                    if (!h3) break;
                    __syncwarp();
                    h2 = fetch(w2, m2);
                    step_merge(w3, m3);
                    if (!h0) break;
                    __syncwarp();
                    h3 = fetch(w3, m3);
                }
            } else {
                for (int t = 0; t < na; ++t) {
                    const SR sr = rec[t];
                    for (int q0 = 0; q0 < sr.len; q0 += 32) {
                        uint32_t w = 0, m = 0;
                        if (q0 + lane < sr.len) load(sr, q0 + lane, w, m);
                        step_or(w, m);
                        __syncwarp();
                    }
                }
            }
            __syncwarp();
        }
        int64_t sn = 0, en = 0;
        if (inext >= 0) {
            sn = ld(arm, inext);
            en = ld(arm, inext + 1);
        }
        cnt = warp_sum(cnt);
        if (lane == 0) counts[i] = cnt;
        __syncwarp();
        if (nt <= PAT_WORDS) {
            // sort the touched words as (word - min) << log2 S | slot, keep the pattern,
            // clear the slots
            constexpr int E = PAT_WORDS / 32;
            uint32_t hsl[E], wd[E];
            uint32_t mn = 0xffffffffu, mx = 0u;
#pragma unroll
            for (int q = 0; q < E; ++q) {
                const int idx = lane * E + q;
                hsl[q] = idx < nt ? wl[idx] : 0u;
                wd[q] = idx < nt ? keys[hsl[q]] : 0u;
                if (idx < nt) {
                    mn = min(mn, wd[q]);
                    mx = max(mx, wd[q]);
                }
            }
            mn = __reduce_min_sync(FULL, mn);
            mx = __reduce_max_sync(FULL, mx);
            const bool packed = nt == 0 || (mx - mn) < ((1u << (32 - LOGS)) - 1u);
            uint32_t v[E];
#pragma unroll
            for (int q = 0; q < E; ++q) {
                const int idx = lane * E + q;
                v[q] = idx < nt ? (((wd[q] - mn) << LOGS) | hsl[q]) : 0xffffffffu;
            }
            if (packed) warp_bitonic_sort<E>(v);
            long long off = -1;
            if (po.pat && packed) {
                if (lane == 0) {
                    const unsigned long long o = atomicAdd(&st->pat_used, (unsigned long long)nt);
                    off = (o + (unsigned long long)nt <= (unsigned long long)po.cap) ? (long long)o : -1;
                }
                off = __shfl_sync(FULL, off, 0);
            }
#pragma unroll
            for (int q = 0; q < E; ++q) {
                const int idx = lane * E + q;
                if (idx < nt) {
                    const uint32_t hs = v[q] & (S - 1);
                    const uint32_t m = masks[hs];
                    const uint32_t w = keys[hs];
                    keys[hs] = EMPTY;
                    masks[hs] = 0;
                    if (off >= 0) po.pat[off + idx] = make_uint2(w, m);
                }
            }
            if (po.pat && lane == 0) {
                po.off[i] = off;
                po.len[i] = nt;
            }
        } else {
            for (int t = lane; t < S; t += 32) {
                keys[t] = EMPTY;
                masks[t] = 0;
            }
        }
        if (inext >= 0) jn = lane < en - sn ? __ldg(aent + sn + lane) : 0;
        __syncwarp();
        if (inext < 0) break;
        r = rn;
        i = inext;
        s = sn;
        e = en;
    }
}

template <typename OffT, int W>
__global__ void __launch_bounds__(256, 1) k_sym_window(const OffT* __restrict__ arm, const int32_t* __restrict__ aent,
                                                    const OffT* __restrict__ brm, const int32_t* __restrict__ bent,
                                                    const int32_t* __restrict__ bc_len,
                                                    const uint2* __restrict__ pairs, const int32_t* __restrict__ perm,
                                                    const int* __restrict__ bin_start, int bin,
                                                    const int32_t* __restrict__ wlo, int32_t* __restrict__ counts,
                                                    PatOut po, DevStatus* st, long long nnzB) {
    constexpr int NW = W / 32;
    constexpr int WB = NW + 672 + PAT_WORDS;  // words per warp: bitmap | recs | flat | scratch | list
    extern __shared__ __align__(16) uint32_t sm_win[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, warps = blockDim.x >> 5;
    uint32_t* bm = sm_win + (size_t)warp * WB;
    void* rec = (void*)(bm + NW);
    uint32_t* wl = bm + NW + 672;
    const int r0 = bin_start[bin], r1 = bin_start[bin + 1];
    if (r0 + blockIdx.x * warps + warp >= r1) return;
    for (int t = lane; t < NW / 4; t += 32) ((uint4*)bm)[t] = make_uint4(0, 0, 0, 0);
    __syncwarp();
    const bool o32 = nnzB < INT32_MAX;
    if (st->use_comp) {
        if (o32)
            sym_window_rows<OffT, W, true, true>(arm, aent, brm, bent, bc_len, pairs, perm, r0, r1, wlo, counts, bm,
                                                 rec, wl, po, st);
        else
            sym_window_rows<OffT, W, true, false>(arm, aent, brm, bent, bc_len, pairs, perm, r0, r1, wlo, counts, bm,
                                                  rec, wl, po, st);
    } else {
        if (o32)
            sym_window_rows<OffT, W, false, true>(arm, aent, brm, bent, bc_len, pairs, perm, r0, r1, wlo, counts, bm,
                                                  rec, wl, po, st);
        else
            sym_window_rows<OffT, W, false, false>(arm, aent, brm, bent, bc_len, pairs, perm, r0, r1, wlo, counts,
                                                   bm, rec, wl, po, st);
    }
}

// ------------------------------------------------------------------------------------
// a5 for window rows, lean form (k_sym_rows): the same bit-vector accumulator (accum = OR,
// PAPER.md:171, 180) and kept pattern as sym_window_rows, without the flattened pairs and
// their duplicate-word merging.  A B_C row has distinct words, so a B_C row per group of
// lanes needs no merging: with B_C rows of <= G pairs, R = 32 / G rows run per warp step
// (G = 8, 10, 16, 32), their bit-vector read-OR-writes in R rounds (rows of a step may share
// words), the counting of new bits and the touched-word list once per step.  Longer rows
// take the whole warp per 32-pair segment.  Pairs are loaded one step ahead.  The
// touched-word list is sorted with one key per lane when it holds <= 32 words.  Pattern
// space is taken from the pool in warp-private blocks (one pool atomic per block of pblk
// pairs, not per row; pblk = the pool share of one warp, clamped to [PAT_WORDS, 2048]).
// Needs B.nnz < 2^31; without B_C (COMP = false, words repeat inside a B row) the OR is a
// shared atomic.
// ------------------------------------------------------------------------------------

// S > 0 (HT): rows whose columns do not fit a window keep their words in a warp-owned hash
// table (keys[S] | masks[S], bank-major linear probing, write-then-verify claims) instead of
// the bit vector; the list holds slots, the epilogue sorts the words and re-finds them.
template <typename OffT, int W, bool COMP, int S>
__device__ __forceinline__ void sym_rows_body(const OffT* __restrict__ arm, const int32_t* __restrict__ aent,
                                              const OffT* __restrict__ brm, const int32_t* __restrict__ bent,
                                              const int32_t* __restrict__ bc_len, const uint2* __restrict__ pairs,
                                              const int32_t* __restrict__ perm, const int* __restrict__ bin_start,
                                              int bin, const int32_t* __restrict__ wlo, int32_t* __restrict__ counts,
                                              PatOut po, DevStatus* st, int pblk, int atom, int* retry) {
    constexpr bool HT = S > 0;
    // speculative HT (retry != null): a small table for rows whose bound ub overstates their
    // distinct words; a row that finds more than S/2 words is abandoned (its remaining steps
    // skipped) and appended to retry[2..] (count in retry[1]) for a full-size table
    const bool spec = HT && retry != nullptr;
    bool over = false;
    constexpr int NW = HT ? 2 * S : W / 32;   // bitmap words, or keys[S] | masks[S]
    constexpr int WB = NW + 64 + PAT_WORDS;  // words per warp: bitmap | rec[32] (int2) | list
    extern __shared__ __align__(16) uint32_t sm_rows[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, warps = blockDim.x >> 5;
    uint32_t* bm = sm_rows + (size_t)warp * WB;
    int2* rec = (int2*)(bm + NW);
    uint32_t* wl = bm + NW + 64;
    const int r0 = bin_start[bin], r1 = bin_start[bin + 1];
    const int stride = gridDim.x * warps;
    int r = r0 + blockIdx.x * warps + warp;
    if (r >= r1) return;
    uint32_t* hkeys = bm;      // HT
    uint32_t* hmask = bm + S;  // HT
    auto clear_all = [&]() {
        if (HT) {
            for (int t = lane; t < S; t += 32) {
                hkeys[t] = EMPTY;
                hmask[t] = 0;
            }
        } else {
            for (int t = lane; t < NW / 4; t += 32) ((uint4*)bm)[t] = make_uint4(0, 0, 0, 0);
        }
    };
    clear_all();
    long long pcur = 0, pend = 0;  // this warp's block of the pattern pool
    auto pair_at = [&](int q) -> uint2 {
        if (COMP) return __ldg(pairs + q);
        const int c = __ldg(bent + q);
        return make_uint2((uint32_t)c >> 5, 1u << (c & 31));
    };
    // rows are software-pipelined: the next row's bounds and window are loaded when a row
    // starts, its first 32 A entries when the row's products are done
    int i = perm[r];
    int64_t s = ld(arm, i), e = ld(arm, i + 1);
    uint32_t wb = HT ? 0u : (uint32_t)__ldg(wlo + i) >> 5;
    int jfirst = lane < e - s ? __ldg(aent + s + lane) : 0;
    int inext = r + stride < r1 ? __ldg(perm + r + stride) : -1;
    __syncwarp();
    while (true) {
        int64_t sn = 0, en = 0;
        uint32_t wbn = 0;
        if (inext >= 0) {
            sn = ld(arm, inext);
            en = ld(arm, inext + 1);
            wbn = HT ? 0u : (uint32_t)__ldg(wlo + inext) >> 5;
        }
        const int inext2 = r + 2 * stride < r1 ? __ldg(perm + r + 2 * stride) : -1;
        int cnt = 0, nt = 0;
        // count the bits a lane added and list the words it turned non-zero (tag: the word's
        // bit-vector index, or its hash slot)
        auto post = [&](uint32_t tag, uint32_t m, uint32_t old, bool act) {
            const bool fresh = act && old == 0;
            if (act) cnt += __popc(m & ~old);
            const unsigned fb = __ballot_sync(FULL, fresh);
            if (fresh) {
                const int pos = nt + __popc(fb & lanemask_lt());
                if (pos < PAT_WORDS) wl[pos] = tag;
            }
            nt += __popc(fb);
            if (spec) over = nt > S / 2;  // warp-uniform; at most S/2 + 32 slots taken
        };
        // OR m into word w for the lanes with act (warp-collective: HT claims slots); returns
        // the old mask, tag = bit-vector index or slot.  PLAIN: the active lanes' words are
        // distinct (one B_C row), else the OR is atomic.
        auto rmw = [&](uint32_t w, uint32_t m, bool act, bool plain, uint32_t& tag) -> uint32_t {
            uint32_t* cell;
            if constexpr (HT) {
                tag = strict_claim<S>(hkeys, w, act);
                cell = hmask + tag;
            } else {
                tag = w - wb;
                cell = bm + tag;
            }
            if (!act) return 0u;
            if (plain) {
                const uint32_t old = *cell;
                *cell = old | m;
                return old;
            }
            return atomicOr(cell, m);
        };
        for (int64_t a0 = s; a0 < e && !over; a0 += 32) {
            const int na = (int)min((int64_t)32, e - a0);
            int bb = 0, bl = 0;
            if (lane < na) {
                const int j = a0 == s ? jfirst : __ldg(aent + a0 + lane);
                bb = (int)ld(brm, j);
                bl = COMP ? __ldg(bc_len + j) : (int)(ld(brm, j + 1) - bb);
            }
            const unsigned ne = __ballot_sync(FULL, bl > 0);
            const int ntr = __popc(ne);
            const int maxbl = (int)__reduce_max_sync(FULL, (unsigned)bl);
            __syncwarp();
            if (bl > 0) rec[__popc(ne & lanemask_lt())] = make_int2(bb, bl);
            __syncwarp();
            if (ntr == 0) continue;
            // R rows per step, G = 32 / R lanes per row (lanes >= R*G idle); loads of the
            // next step are unconditional (indices clamped into the chunk's last row)
            auto run = [&](auto RC) {
                constexpr int R = decltype(RC)::value;
                constexpr int G = 32 / R;
                const int grp = lane / G, gl = lane - grp * G;
                auto fetch = [&](int t, uint2& p, bool& act) {
                    const int tt = t + grp;
                    const int2 rr = rec[min(tt, ntr - 1)];
                    act = grp < R && tt < ntr && gl < rr.y;
                    p = pair_at(rr.x + min(gl, rr.y - 1));
                };
                uint2 p;
                bool act;
                fetch(0, p, act);
                for (int t = 0; t < ntr && !over; t += R) {
                    uint2 pn;
                    bool actn;
                    fetch(t + R, pn, actn);
                    uint32_t old = 0, tag = 0;
                    if (COMP && !HT && atom) {
                        // all R rows in one round of shared atomic ORs: lanes sharing a word
                        // are ordered by the atomics, so each new bit is counted once and
                        // exactly one lane sees the word's old mask as 0 (default)
                        old = rmw(p.x, p.y, act, false, tag);
                        __syncwarp();
                    } else if (COMP) {
                        // rows of a step may share words: one row per round
#pragma unroll
                        for (int k = 0; k < R; ++k) {
                            uint32_t tg;
                            const uint32_t o = rmw(p.x, p.y, act && grp == k, true, tg);
                            if (act && grp == k) {
                                old = o;
                                tag = tg;
                            }
                            __syncwarp();
                        }
                    } else {
                        old = rmw(p.x, p.y, act, false, tag);
                        __syncwarp();
                    }
                    post(tag, p.y, old, act);
                    p = pn;
                    act = actn;
                }
            };
            if (COMP && atom && maxbl <= 32) {
                // the chunk's B_C rows back to back, 32 pairs per step: one round of atomic ORs
                // per step (lanes of different rows sharing a word are ordered by the atomics),
                // no lanes idle past the end of short rows.  Row of flat pair f: the rows that
                // start in the step's window are one OR-reduction of their start bits; a lane's
                // row is the count of those at or below it (rows are non-empty, so starts are
                // distinct).  Pairs are loaded one step ahead.
                int pex = lane < ntr ? rec[lane].y : 0;
#pragma unroll
                for (int d = 1; d < 32; d <<= 1) {
                    const int y = __shfl_up_sync(FULL, pex, d);
                    if (lane >= d) pex += y;
                }
                const int T = __shfl_sync(FULL, pex, 31);
                pex -= lane < ntr ? rec[lane].y : 0;  // exclusive prefix: first pair of row lane
                int cur = -1;
                auto fetch = [&](int f0, uint2& p, bool& act) {
                    const unsigned M = __reduce_or_sync(
                        FULL, (lane < ntr && pex >= f0 && pex < f0 + 32) ? 1u << (pex - f0) : 0u);
                    const int t = min(max(cur + __popc(M & lanemask_le()), 0), ntr - 1);
                    cur += __popc(M);
                    const int2 rr = rec[t];
                    const int f = f0 + lane;
                    act = f < T;
                    const int off = min(f - __shfl_sync(FULL, pex, t), rr.y - 1);
                    p = pair_at(rr.x + max(off, 0));
                };
                uint2 p;
                bool act;
                fetch(0, p, act);
                for (int f0 = 0; f0 < T && !over; f0 += 32) {
                    uint2 pn = p;
                    bool actn = false;
                    if (f0 + 32 < T) fetch(f0 + 32, pn, actn);
                    uint32_t tag = 0;
                    const uint32_t old = rmw(p.x, p.y, act, false, tag);
                    __syncwarp();
                    post(tag, p.y, old, act);
                    p = pn;
                    act = actn;
                }
            } else if (maxbl <= 8)
                run(std::integral_constant<int, 4>{});
            else if (maxbl <= 10)
                run(std::integral_constant<int, 3>{});
            else if (maxbl <= 16)
                run(std::integral_constant<int, 2>{});
            else if (maxbl <= 32)
                run(std::integral_constant<int, 1>{});
            else {
                for (int t = 0; t < ntr && !over; ++t) {
                    const int2 rr = rec[t];
                    for (int q0 = 0; q0 < rr.y && !over; q0 += 32) {
                        const bool act = q0 + lane < rr.y;
                        const uint2 pq = pair_at(rr.x + min(q0 + lane, rr.y - 1));
                        uint32_t tag;
                        const uint32_t old = rmw(pq.x, pq.y, act, COMP, tag);
                        post(tag, pq.y, old, act);
                        __syncwarp();
                    }
                }
            }
            __syncwarp();
        }
        jfirst = inext >= 0 && lane < en - sn ? __ldg(aent + sn + lane) : 0;
        cnt = warp_sum(cnt);
        if (over) {
            // abandoned: to the retry list, table cleared
            if (lane == 0) retry[2 + atomicAdd(&retry[1], 1)] = i;
            clear_all();
        } else if (lane == 0) {
            counts[i] = cnt;
        }
        __syncwarp();
        if (over) {
            over = false;
        } else if (nt <= PAT_WORDS) {
            // sorted pattern into the pool, clear the listed words
            long long off = -1;
            if (po.pat) {
                if (pcur + nt > pend) {
                    long long o = 0;
                    if (lane == 0) o = (long long)atomicAdd(&st->pat_used, (unsigned long long)pblk);
                    o = __shfl_sync(FULL, o, 0);
                    pcur = o;
                    pend = min(o + pblk, (long long)po.cap);
                }
                if (pcur + nt <= pend) {
                    off = pcur;
                    pcur += nt;
                }
            }
            if (HT) {
                // sort the listed words, re-find their slots, then clear them
                uint32_t v[2];
#pragma unroll
                for (int q = 0; q < 2; ++q) v[q] = lane * 2 + q < nt ? hkeys[wl[lane * 2 + q]] : 0xffffffffu;
                warp_bitonic_sort<2>(v);
                uint32_t sl[2] = {0u, 0u};
#pragma unroll
                for (int q = 0; q < 2; ++q) {
                    const int idx = lane * 2 + q;
                    if (idx < nt) {
                        sl[q] = strict_find<S>(hkeys, v[q]);
                        if (off >= 0) po.pat[off + idx] = make_uint2(v[q], hmask[sl[q]]);
                    }
                }
                __syncwarp();
#pragma unroll
                for (int q = 0; q < 2; ++q) {
                    if (lane * 2 + q < nt) {
                        hkeys[sl[q]] = EMPTY;
                        hmask[sl[q]] = 0;
                    }
                }
            } else if (nt <= 32) {
                uint32_t v[1] = {lane < nt ? wl[lane] : 0xffffffffu};
                warp_bitonic_sort<1>(v);
                if (lane < nt) {
                    const uint32_t m = bm[v[0]];
                    bm[v[0]] = 0;
                    if (off >= 0) po.pat[off + lane] = make_uint2(v[0] + wb, m);
                }
            } else {
                uint32_t v[2];
#pragma unroll
                for (int q = 0; q < 2; ++q) v[q] = lane * 2 + q < nt ? wl[lane * 2 + q] : 0xffffffffu;
                warp_bitonic_sort<2>(v);
#pragma unroll
                for (int q = 0; q < 2; ++q) {
                    const int idx = lane * 2 + q;
                    if (idx < nt) {
                        const uint32_t m = bm[v[q]];
                        bm[v[q]] = 0;
                        if (off >= 0) po.pat[off + idx] = make_uint2(v[q] + wb, m);
                    }
                }
            }
            if (po.pat && lane == 0) {
                po.off[i] = off;
                po.len[i] = nt;
            }
        } else {
            clear_all();
        }
        __syncwarp();
        if (inext < 0) break;
        r += stride;
        i = inext;
        s = sn;
        e = en;
        wb = wbn;
        inext = inext2;
    }
}

// one launch for both compression modes (decided on the device in a1): the body is
// instantiated for B_C pairs and for plain B entries
template <typename OffT, int W, int S = 0>
__global__ void __launch_bounds__(256, S == 0 ? 4 : 1) k_sym_rows(const OffT* __restrict__ arm, const int32_t* __restrict__ aent,
                                                  const OffT* __restrict__ brm, const int32_t* __restrict__ bent,
                                                  const int32_t* __restrict__ bc_len,
                                                  const uint2* __restrict__ pairs, const int32_t* __restrict__ perm,
                                                  const int* __restrict__ bin_start, int bin,
                                                  const int32_t* __restrict__ wlo, int32_t* __restrict__ counts,
                                                  PatOut po, DevStatus* st, int pblk, int atom, int* retry) {
    if (st->use_comp)
        sym_rows_body<OffT, W, true, S>(arm, aent, brm, bent, bc_len, pairs, perm, bin_start, bin, wlo, counts, po, st,
                                        pblk, atom, retry);
    else
        sym_rows_body<OffT, W, false, S>(arm, aent, brm, bent, bc_len, pairs, perm, bin_start, bin, wlo, counts, po,
                                         st, pblk, atom, retry);
}

// KK_SYM_ROWS=0 selects k_sym_window for the window bins (experiments)
static bool use_sym_rows() {
    static const bool v = [] {
        const char* s = getenv("KK_SYM_ROWS");
        return !(s && s[0] == '0');
    }();
    return v;
}

// KK_SYM_SPEC=0 disables the speculative small tables (experiments)
static bool sym_spec() {
    const char* s = getenv("KK_SYM_SPEC");
    return !(s && s[0] == '0');
}

// Window rows take a step's B_C rows in one round of shared atomic ORs (C2 sym_rows 1.13
// -> 1.04 ms against one plain read-OR-write round per row)
static int sym_atom() { return 1; }

template <typename OffT, int W>
static void launch_sym_rows(Launch& L, const SymArgs& a, int bin) {
    const int warps = W <= 65536 ? 8 : 4;  // 128K/192K-bit windows: 16/24 KB per warp
    const size_t smem = (size_t)warps * ((size_t)W / 32 + 64 + PAT_WORDS) * 4;
    auto kern = k_sym_rows<OffT, W>;
    KCfg c = kernel_cfg(kern, warps * 32, smem, L.num_sms);
    const int64_t hr = host_rows(a, bin);
    if (hr == 0) return;
    int64_t need = ((hr > 0 ? hr : a.A.nrows) + warps - 1) / warps;
    int grid = (int)std::min<int64_t>(need, c.grid_cap);
    const int64_t share = a.pat.cap / ((int64_t)grid * warps);
    const int pblk = (int)std::max<int64_t>(PAT_WORDS, std::min<int64_t>(2048, share));
    L.begin(kname("sym_rows", W), L.stream);
    kern<<<grid, warps * 32, smem, L.stream>>>((const OffT*)a.A.row_map, a.A.entries, (const OffT*)a.B.row_map,
                                               a.B.entries, a.bc_len, a.pairs, a.perm, a.bin_start, bin, a.wlo,
                                               a.counts, a.pat, (DevStatus*)a.st, pblk, sym_atom(), nullptr);
    L.end(L.stream);
}

template <typename OffT, int W>
static void launch_sym_window(Launch& L, const SymArgs& a, int bin) {
    if (a.B.nnz < INT32_MAX && use_sym_rows()) {
        launch_sym_rows<OffT, W>(L, a, bin);
        return;
    }
    const int warps = W <= 16384 ? 8 : 4;
    const size_t smem = (size_t)warps * ((size_t)W / 32 + 672 + PAT_WORDS) * 4;
    auto kern = k_sym_window<OffT, W>;
    KCfg c = kernel_cfg(kern, warps * 32, smem, L.num_sms);
    int64_t need = (a.A.nrows + warps - 1) / warps;
    int grid = (int)std::min<int64_t>(need, c.grid_cap);
    L.begin(kname("sym_window", W), L.stream);
    kern<<<grid, warps * 32, smem, L.stream>>>((const OffT*)a.A.row_map, a.A.entries, (const OffT*)a.B.row_map,
                                               a.B.entries, a.bc_len, a.pairs, a.perm, a.bin_start, bin, a.wlo,
                                               a.counts, a.pat, (DevStatus*)a.st, (long long)a.B.nnz);
    L.end(L.stream);
}

template <typename OffT, int S>
__global__ void __launch_bounds__(256, 1) k_sym_hash(const OffT* __restrict__ arm, const int32_t* __restrict__ aent,
                                                     const OffT* __restrict__ brm, const int32_t* __restrict__ bent,
                                                     const int32_t* __restrict__ bc_len, const uint2* __restrict__ pairs,
                                                     const int32_t* __restrict__ perm, const int* __restrict__ bin_start,
                                                     int bin, int32_t* __restrict__ counts, PatOut po, DevStatus* st,
                                                     long long nnzB) {
    constexpr int WB = 2 * S + 672 + PAT_WORDS;  // words per warp: keys | masks | recs | flat | scratch | list
    extern __shared__ __align__(16) uint32_t sm_hs[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, warps = blockDim.x >> 5;
    uint32_t* keys = sm_hs + (size_t)warp * WB;
    uint32_t* masks = keys + S;
    void* rec = (void*)(masks + S);
    uint32_t* wl = masks + S + 672;
    const int r0 = bin_start[bin], r1 = bin_start[bin + 1];
    if (r0 + blockIdx.x * warps + warp >= r1) return;
    for (int t = lane; t < S; t += 32) {
        keys[t] = EMPTY;
        masks[t] = 0;
    }
    __syncwarp();
    const bool o32 = nnzB < INT32_MAX;
    if (st->use_comp) {
        if (o32)
            sym_hash_rows<OffT, S, true, true>(arm, aent, brm, bent, bc_len, pairs, perm, r0, r1, counts, keys, masks,
                                               rec, wl, po, st);
        else
            sym_hash_rows<OffT, S, true, false>(arm, aent, brm, bent, bc_len, pairs, perm, r0, r1, counts, keys, masks,
                                                rec, wl, po, st);
    } else {
        if (o32)
            sym_hash_rows<OffT, S, false, true>(arm, aent, brm, bent, bc_len, pairs, perm, r0, r1, counts, keys, masks,
                                                rec, wl, po, st);
        else
            sym_hash_rows<OffT, S, false, false>(arm, aent, brm, bent, bc_len, pairs, perm, r0, r1, counts, keys,
                                                 masks, rec, wl, po, st);
    }
}

// retry: speculative launch (rows abandoned past S/2 words go to the list); list: the
// retry list as the bin (perm = list + 2, bin_start = list, bin 0; row count unknown on the host)
template <typename OffT, int S>
static void launch_sym_rows_ht(Launch& L, const SymArgs& a, int bin, int* retry = nullptr, int* list = nullptr) {
    const int warps = S <= 1024 ? 8 : (S <= 2048 ? 4 : 2);
    const size_t smem = (size_t)warps * ((size_t)2 * S + 64 + PAT_WORDS) * 4;
    auto kern = k_sym_rows<OffT, 32, S>;
    KCfg c = kernel_cfg(kern, warps * 32, smem, L.num_sms);
    const int64_t hr = host_rows(a, bin);  // list: at most the bin's rows come back
    if (hr == 0) return;
    int64_t need = ((hr > 0 ? hr : a.A.nrows) + warps - 1) / warps;
    int grid = (int)std::min<int64_t>(need, c.grid_cap);
    const int64_t share = a.pat.cap / ((int64_t)grid * warps);
    const int pblk = (int)std::max<int64_t>(PAT_WORDS, std::min<int64_t>(2048, share));
    L.begin(list ? kname("sym_rows_retry", S) : retry ? kname("sym_rows_spec", S) : kname("sym_rows_ht", S), L.stream);
    kern<<<grid, warps * 32, smem, L.stream>>>((const OffT*)a.A.row_map, a.A.entries, (const OffT*)a.B.row_map,
                                               a.B.entries, a.bc_len, a.pairs, list ? list + 2 : a.perm,
                                               list ? list : a.bin_start, list ? 0 : bin, a.wlo, a.counts, a.pat,
                                               (DevStatus*)a.st, pblk, sym_atom(), retry);
    L.end(L.stream);
}

// hash bins: rows with ub <= cap = 64 << (bin - 1) words; table S = 2 * cap
template <typename OffT, int S>
static void launch_sym_hash(Launch& L, const SymArgs& a, int bin) {
    if (a.B.nnz < INT32_MAX && use_sym_rows()) {
        launch_sym_rows_ht<OffT, S>(L, a, bin);
        return;
    }
    const int warps = S <= 1024 ? 8 : (S <= 4096 ? 4 : 2);
    const size_t smem = (size_t)warps * (2 * S + 672 + PAT_WORDS) * 4;
    auto kern = k_sym_hash<OffT, S>;
    KCfg c = kernel_cfg(kern, warps * 32, smem, L.num_sms);
    int64_t need = (a.A.nrows + warps - 1) / warps;
    int grid = (int)std::min<int64_t>(need, c.grid_cap);
    L.begin(kname("sym_hash", S), L.stream);
    kern<<<grid, warps * 32, smem, L.stream>>>((const OffT*)a.A.row_map, a.A.entries, (const OffT*)a.B.row_map,
                                               a.B.entries, a.bc_len, a.pairs, a.perm, a.bin_start, bin, a.counts,
                                               a.pat, (DevStatus*)a.st, (long long)a.B.nnz);
    L.end(L.stream);
}

// a5 for tiny rows (flops_i <= TINY_MAX): a lane owns a row; its distinct columns in a
// register list (TinyList; the paper's accumulator in K registers, accum = set insert)
template <typename OffT>
__global__ void __launch_bounds__(256) k_sym_tiny(const OffT* __restrict__ arm, const int32_t* __restrict__ aent,
                                                  const OffT* __restrict__ brm, const int32_t* __restrict__ bent,
                                                  const int32_t* __restrict__ perm, const int* __restrict__ bin_start,
                                                  int bin, int32_t* __restrict__ counts) {
    const int r0 = bin_start[bin], r1 = bin_start[bin + 1];
    for (int r = r0 + blockIdx.x * blockDim.x + threadIdx.x; r < r1; r += gridDim.x * blockDim.x) {
        const int i = perm[r];
        TinyList<TINY_MAX, float, false> T;
        const int64_t s = ld(arm, i), e = ld(arm, i + 1);
        for (int64_t p = s; p < e; ++p) {
            const int j = __ldg(aent + p);
            const int64_t bs = ld(brm, j), be = ld(brm, j + 1);
            for (int64_t q = bs; q < be; ++q) T.insert(__ldg(bent + q), 0.0f);
        }
        counts[i] = T.n;
    }
}

template <typename OffT>
static void launch_sym_tiny(Launch& L, const SymArgs& a) {
    const int64_t hr = host_rows(a, SYM_TINY_BIN);
    if (hr == 0) return;
    auto kern = k_sym_tiny<OffT>;
    KCfg c = kernel_cfg(kern, 256, 0, L.num_sms);
    const int grid = (int)std::min<int64_t>(((hr > 0 ? hr : a.A.nrows) + 255) / 256, c.grid_cap);
    L.begin("sym_tiny", L.stream);
    kern<<<grid, 256, 0, L.stream>>>((const OffT*)a.A.row_map, a.A.entries, (const OffT*)a.B.row_map, a.B.entries,
                                     a.perm, a.bin_start, SYM_TINY_BIN, a.counts);
    L.end(L.stream);
}

template <typename OffT>
static void symbolic_bins_t(Launch& L, const SymArgs& a, cudaStream_t dense_stream) {
    // dense rows first (heaviest), on their own stream when given
    const int64_t hdense = host_rows(a, SYM_DENSE_BIN);
    if (hdense != 0) {
        const int threads = 1024;
        int64_t wbits = 200 * 1024 * 8;  // 200 KB bit vector
        const int64_t k32 = ((a.k + 31) / 32) * 32;
        if (k32 < wbits) wbits = k32 > 0 ? k32 : 32;
        const size_t smem = (size_t)(wbits / 8) + 1025 * 4;  // + the long-entry list
        auto kern = k_sym_dense<OffT>;
        KCfg c = kernel_cfg(kern, threads, smem, L.num_sms);
        cudaStream_t s = dense_stream ? dense_stream : L.stream;
        L.begin("sym_dense", s);
        const int grid = (int)(hdense > 0 ? std::min<int64_t>(hdense, c.grid_cap) : c.grid_cap);
        kern<<<grid, threads, smem, s>>>((const OffT*)a.A.row_map, a.A.entries, (const OffT*)a.B.row_map,
                                               a.B.entries, a.bc_len, a.pairs, a.perm, a.bin_start, SYM_DENSE_BIN,
                                               a.k, wbits, a.cursors, a.counts, a.st);
        L.end(s);
    }
    launch_sym_tiny<OffT>(L, a);
    launch_sym_window<OffT, 196608>(L, a, SYM_WIN_BIN0 + 6);
    launch_sym_window<OffT, 131072>(L, a, SYM_WIN_BIN0 + 5);
    launch_sym_window<OffT, 65536>(L, a, SYM_WIN_BIN0 + 4);
    launch_sym_window<OffT, 49152>(L, a, SYM_WIN_BIN0 + 3);
    launch_sym_window<OffT, 32768>(L, a, SYM_WIN_BIN0 + 2);
    launch_sym_window<OffT, 16384>(L, a, SYM_WIN_BIN0 + 1);
    launch_sym_window<OffT, 8192>(L, a, SYM_WIN_BIN0);
    if (a.logG >= 3 && a.retry && a.host_bin_start && a.B.nnz < INT32_MAX && use_sym_rows() && sym_spec()) {
        // rows bound for the large tables (ub > 512 words) first try a 256-slot table: the
        // bound (sum of their B_C rows' lengths) overstates the distinct words of rows whose
        // B rows overlap (C5: ~40 words against ub ~1,000); rows past 128 words are redone
        // with the largest table from the retry list
        // per-bin retry lists (list b at retry + off_b: {0, count, rows...}), so a row that
        // gives up is redone with its own bin's table
        int64_t off[8] = {0};
        int64_t o = 0;
        for (int b = 4; b <= 7; ++b) {
            off[b] = o;
            o += (host_rows(a, b) > 0 ? host_rows(a, b) : 0) + 2;
        }
        cudaMemsetAsync(a.retry, 0, (size_t)o * sizeof(int), L.stream);
        for (int b = 7; b >= 4; --b)
            if (host_rows(a, b) != 0) launch_sym_rows_ht<OffT, 256>(L, a, b, a.retry + off[b]);
        if (host_rows(a, 7) != 0) launch_sym_rows_ht<OffT, 8192>(L, a, 7, nullptr, a.retry + off[7]);
        if (host_rows(a, 6) != 0) launch_sym_rows_ht<OffT, 4096>(L, a, 6, nullptr, a.retry + off[6]);
        if (host_rows(a, 5) != 0) launch_sym_rows_ht<OffT, 2048>(L, a, 5, nullptr, a.retry + off[5]);
        if (host_rows(a, 4) != 0) launch_sym_rows_ht<OffT, 1024>(L, a, 4, nullptr, a.retry + off[4]);
        launch_sym_hash<OffT, 512>(L, a, 3);
        launch_sym_hash<OffT, 256>(L, a, 2);
        launch_sym_hash<OffT, 128>(L, a, 1);
    } else if (a.logG >= 3) {
        // B rows of >= ~5 words on average: flattened-pair hash kernels (keep patterns)
        launch_sym_hash<OffT, 8192>(L, a, 7);
        launch_sym_hash<OffT, 4096>(L, a, 6);
        launch_sym_hash<OffT, 2048>(L, a, 5);
        launch_sym_hash<OffT, 1024>(L, a, 4);
        launch_sym_hash<OffT, 512>(L, a, 3);
        launch_sym_hash<OffT, 256>(L, a, 2);
        launch_sym_hash<OffT, 128>(L, a, 1);
    } else {
        // very short B rows (e.g. a prolongator): sub-warp groups, several B rows per step
        launch_sym_warp<OffT, 4096>(L, a, 7);
        launch_sym_warp<OffT, 2048>(L, a, 6);
        launch_sym_warp<OffT, 1024>(L, a, 5);
        launch_sym_warp<OffT, 512>(L, a, 4);
        launch_sym_warp<OffT, 256>(L, a, 3);
        launch_sym_warp<OffT, 128>(L, a, 2);
        launch_sym_warp<OffT, 64>(L, a, 1);
    }
}

void symbolic_bins(Launch& L, const SymArgs& a, cudaStream_t dense_stream) {
    if (a.A.nrows == 0) return;
    if (a.off64)
        symbolic_bins_t<int64_t>(L, a, dense_stream);
    else
        symbolic_bins_t<int32_t>(L, a, dense_stream);
}

}  // namespace kk

// kk_numeric.cu -- a7 + a8: numeric phase (Eq. 1, 174, 178) with fused row sort
// (PAPER.md:621-647).
#include "kk_device.cuh"

#include <cstdlib>

namespace kk {
// ------------------------------------------------------------------------------------
// a7: numeric, warp-owned shared hash (accum = +).  With G = 32
// lanes on one strictly increasing B row the keys of a step are distinct, so values
// are updated with plain shared loads/stores; otherwise with shared atomicAdd.
// The compaction is followed by the fused per-row sort (a8) and a coalesced write.
// ------------------------------------------------------------------------------------
template <typename OffT, typename ValT, int S, bool SORT>
__global__ void __launch_bounds__(256, 1) k_num_warp(const OffT* __restrict__ arm, const int32_t* __restrict__ aent,
                                                  const ValT* __restrict__ aval, const OffT* __restrict__ brm,
                                                  const int32_t* __restrict__ bent, const ValT* __restrict__ bval,
                                                  const OffT* __restrict__ crm, int32_t* __restrict__ cent,
                                                  ValT* __restrict__ cval, const int32_t* __restrict__ perm,
                                                  const int* __restrict__ bin_start, int bin, int logG,
                                                  const DevStatus* __restrict__ st, const ValT* __restrict__ dinv,
                                                  double omega) {
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
        if (dinv) {
            // Jacobi-fused row: C(i,:) = B(i,:) - omega D^-1(i) E(i,:)
            const ValT sc = (ValT)(-omega * (double)__ldg(dinv + i));
            for (int t = lane; t < S; t += 32) vals[t] *= sc;
            __syncwarp();
            const int64_t bs = ld(brm, i), be = ld(brm, i + 1);
            for (int64_t q = bs + lane; q < be; q += 32) {
                bool fresh;
                const uint32_t h = probe_claim<S>(keys, (uint32_t)__ldg(bent + q), &fresh);
                atomicAdd(&vals[h], __ldg(bval + q));
            }
            __syncwarp();
        }
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


// ------------------------------------------------------------------------------------
// a7 (strict B): numeric, warp-owned shared hash with atomic-free claims.
//
// Used when every row of B is strictly increasing (checked in a4), so the <= 32 products
// of one warp step -- 32 consecutive entries of ONE B row -- have distinct keys:
//   * claims use write-then-verify (a lane writes its key into an EMPTY slot, the warp
//     syncs, the lane re-reads; one writer wins, the others probe on) -- no ATOMS.CAS;
//   * values are updated with a plain shared load / add / store (slots are distinct).
// Slot layout is bank-major: probe position L in [0,S) maps to slot (L % R)*32 + L / R
// (R = S/32 rows of 32 banks), and a key starts at L0 = (col & 31)*R + hash(col >> 5),
// so keys of consecutive columns sit in different banks (stencil rows are runs of
// consecutive columns) and a probe sequence stays in its bank until the bank is full.
// The A row is staged per 32-entry chunk in shared memory (B row start/length, a_ij),
// and the B row of the next step is loaded while the current step is inserted.
// Epilogue (a8): compaction by ballot into (col - cmin) << log2(S) | slot, a warp bitonic
// sort of those 32-bit words in registers, coalesced writes, and the table is reset at
// exactly the slots that were used.
// ------------------------------------------------------------------------------------
// Per A entry of the current 32-entry chunk: its B row (start, length) and a_ij, read back
// per step with one (O32: element offsets < 2^31) or two 16-byte shared loads.
template <typename ValT, bool O32>
struct StepRec;
template <typename ValT>
struct __align__(16) StepRec<ValT, true> {
    int bb;
    int len;
    double a;
};
template <typename ValT>
struct __align__(16) StepRec<ValT, false> {
    long long bb;
    int len;
    int pad;
    double a;
    double pad2;
};
constexpr size_t REC_BYTES = 32 * 32;  // room for 32 records of either kind

// Shared-memory layout of one warp: vals[S] | rec[32] | keys[S] | stage[CAP]
template <typename ValT, int S, int CAP>
struct StrictLayout {
    static constexpr size_t vals = 0;
    static constexpr size_t rec = ((size_t)S * sizeof(ValT) + 15) / 16 * 16;
    static constexpr size_t keys = rec + REC_BYTES;
    static constexpr size_t stage = keys + (size_t)S * 4;
    static constexpr size_t bytes = (stage + (size_t)CAP * 4 + 15) / 16 * 16;
};

// The products of one row, one B row (or 32-entry segment of it) per warp step, the
// steps in A-entry order: the A row is staged per 32-entry chunk (StepRec per entry),
// the first chunk's A entries (jn, an) come from the caller (prefetched), and B rows are
// loaded three steps ahead of the step being inserted.  insert(col, a_ij * b_jk) is
// called by all 32 lanes for every step (col = EMPTY on idle lanes); the <= 32 columns
// of a step are the entries of one B row segment.
template <typename OffT, typename ValT, bool O32, typename Ins>
__device__ __forceinline__ void row_products(int64_t s, int64_t e, int jn, ValT an, const int32_t* __restrict__ aent,
                                             const ValT* __restrict__ aval, const OffT* __restrict__ brm,
                                             const int32_t* __restrict__ bent, const ValT* __restrict__ bval,
                                             void* rec_raw, Ins insert) {
    using R = StepRec<ValT, O32>;
    R* rec = (R*)rec_raw;
    const int lane = threadIdx.x & 31;
    for (int64_t c0 = s; c0 < e; c0 += 32) {
        const int na = (int)min((int64_t)32, e - c0);
        int j = jn;
        ValT a = an;
        if (c0 != s && lane < na) {
            j = __ldg(aent + c0 + lane);
            a = __ldg(aval + c0 + lane);
        }
        int bl = 0;
        __syncwarp();
        if (lane < na) {
            const int64_t bb = ld(brm, j);
            bl = (int)(ld(brm, j + 1) - bb);
            R sr;
            sr.bb = (decltype(sr.bb))bb;
            sr.len = bl;
            sr.a = (double)a;
            rec[lane] = sr;
        }
        const int maxbl = (int)__reduce_max_sync(FULL, (unsigned)bl);
        __syncwarp();
        if (maxbl == 0) continue;
        // steps in A-entry order; loads run three steps ahead; the product is formed at
        // insert time so no load is waited on early.  `step` fills one step's (col, b)
        // and returns false after the last step.
        auto ring = [&](auto&& step) {
            uint32_t k0, k1, k2, k3;
            ValT b0, b1, b2, b3, a0, a1, a2, a3;
            step(k0, b0, a0);
            bool h1 = step(k1, b1, a1);
            bool h2 = step(k2, b2, a2);
            bool h3 = step(k3, b3, a3);
            while (true) {
                insert(k0, a0 * b0);
                if (!h1) break;
                const bool h0 = step(k0, b0, a0);
                insert(k1, a1 * b1);
                if (!h2) break;
                h1 = step(k1, b1, a1);
                insert(k2, a2 * b2);
                if (!h3) break;
                h2 = step(k2, b2, a2);
                insert(k3, a3 * b3);
                if (!h0) break;
                h3 = step(k3, b3, a3);
            }
        };
        int t = 0;
        if (maxbl <= 32) {
            // one step per A entry (empty B rows give idle steps)
            ring([&](uint32_t& col, ValT& bv, ValT& at) {
                col = EMPTY;
                bv = (ValT)0;
                at = (ValT)0;
                if (t >= na) return false;
                const R sr = rec[t++];
                at = (ValT)sr.a;
                if (lane < sr.len) {
                    col = (uint32_t)__ldg(bent + (sr.bb + lane));
                    bv = __ldg(bval + (sr.bb + lane));
                }
                return true;
            });
        } else {
            // long B rows: steps are (A entry t, 32-entry segment q0 of its B row)
            int q0 = 0;
            while (t < na && rec[t].len == 0) ++t;
            ring([&](uint32_t& col, ValT& bv, ValT& at) {
                col = EMPTY;
                bv = (ValT)0;
                at = (ValT)0;
                if (t >= na) return false;
                const R sr = rec[t];
                at = (ValT)sr.a;
                if (q0 + lane < sr.len) {
                    col = (uint32_t)__ldg(bent + (sr.bb + q0 + lane));
                    bv = __ldg(bval + (sr.bb + q0 + lane));
                }
                q0 += 32;
                if (q0 >= sr.len) {
                    q0 = 0;
                    ++t;
                    while (t < na && rec[t].len == 0) ++t;
                }
                return true;
            });
        }
        __syncwarp();
    }
}

// As row_products, two B rows per warp step: insert2(col0, a*b0, col1, a*b1) gets the
// products of B rows t (col0) and t+1 (col1).  Columns repeat between the two rows, so
// callers must update row t's products before row t+1's.  Loads run two steps (four B
// rows) ahead.
template <typename OffT, typename ValT, bool O32, typename Ins2>
__device__ __forceinline__ void row_products2(int64_t s, int64_t e, int jn, ValT an, const int32_t* __restrict__ aent,
                                              const ValT* __restrict__ aval, const OffT* __restrict__ brm,
                                              const int32_t* __restrict__ bent, const ValT* __restrict__ bval,
                                              void* rec_raw, Ins2 insert2) {
    using R = StepRec<ValT, O32>;
    R* rec = (R*)rec_raw;
    const int lane = threadIdx.x & 31;
    for (int64_t c0 = s; c0 < e; c0 += 32) {
        const int na = (int)min((int64_t)32, e - c0);
        int j = jn;
        ValT a = an;
        if (c0 != s && lane < na) {
            j = __ldg(aent + c0 + lane);
            a = __ldg(aval + c0 + lane);
        }
        int bl = 0;
        __syncwarp();
        if (lane < na) {
            const int64_t bb = ld(brm, j);
            bl = (int)(ld(brm, j + 1) - bb);
            R sr;
            sr.bb = (decltype(sr.bb))bb;
            sr.len = bl;
            sr.a = (double)a;
            rec[lane] = sr;
        }
        const int maxbl = (int)__reduce_max_sync(FULL, (unsigned)bl);
        __syncwarp();
        if (maxbl == 0) continue;
        if (maxbl <= 32) {
            int t = 0;
            auto fetch = [&](uint32_t& c0_, ValT& b0_, ValT& a0_, uint32_t& c1_, ValT& b1_, ValT& a1_) {
                c0_ = c1_ = EMPTY;
                b0_ = b1_ = a0_ = a1_ = (ValT)0;
                if (t >= na) return false;
                const R r0 = rec[t];
                a0_ = (ValT)r0.a;
                if (lane < r0.len) {
                    c0_ = (uint32_t)__ldg(bent + (r0.bb + lane));
                    b0_ = __ldg(bval + (r0.bb + lane));
                }
                if (t + 1 < na) {
                    const R r1 = rec[t + 1];
                    a1_ = (ValT)r1.a;
                    if (lane < r1.len) {
                        c1_ = (uint32_t)__ldg(bent + (r1.bb + lane));
                        b1_ = __ldg(bval + (r1.bb + lane));
                    }
                }
                t += 2;
                return true;
            };
            uint32_t xc0, xc1, yc0, yc1;
            ValT xb0, xb1, xa0, xa1, yb0, yb1, ya0, ya1;
            fetch(xc0, xb0, xa0, xc1, xb1, xa1);
            bool hy = fetch(yc0, yb0, ya0, yc1, yb1, ya1);
            while (true) {
                insert2(xc0, xa0 * xb0, xc1, xa1 * xb1);
                if (!hy) break;
                const bool hx = fetch(xc0, xb0, xa0, xc1, xb1, xa1);
                insert2(yc0, ya0 * yb0, yc1, ya1 * yb1);
                if (!hx) break;
                hy = fetch(yc0, yb0, ya0, yc1, yb1, ya1);
            }
        } else {
            // long B rows: 32-entry segments, one per step
            for (int t = 0; t < na; ++t) {
                const R sr = rec[t];
                const ValT at = (ValT)sr.a;
                for (int q0 = 0; q0 < sr.len; q0 += 32) {
                    uint32_t col = EMPTY;
                    ValT p = (ValT)0;
                    if (q0 + lane < sr.len) {
                        col = (uint32_t)__ldg(bent + (sr.bb + q0 + lane));
                        p = at * __ldg(bval + (sr.bb + q0 + lane));
                    }
                    insert2(col, p, EMPTY, (ValT)0);
                }
            }
        }
        __syncwarp();
    }
}

template <typename OffT, typename ValT, int S, int CAP, bool SORT, bool O32>
__global__ void __launch_bounds__(256, 1) k_num_strict(const OffT* __restrict__ arm, const int32_t* __restrict__ aent,
                                                    const ValT* __restrict__ aval, const OffT* __restrict__ brm,
                                                    const int32_t* __restrict__ bent, const ValT* __restrict__ bval,
                                                    const OffT* __restrict__ crm, int32_t* __restrict__ cent,
                                                    ValT* __restrict__ cval, const int32_t* __restrict__ perm,
                                                    const int* __restrict__ bin_start, int bin,
                                                    const ValT* __restrict__ dinv, double omega) {
    using LY = StrictLayout<ValT, S, CAP>;
    constexpr int LOGS = ilog2(S);
    constexpr int E = CAP / 32;  // sort elements per lane
    extern __shared__ __align__(16) unsigned char sm_num[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, warps = blockDim.x >> 5;
    unsigned char* base = sm_num + (size_t)warp * LY::bytes;
    ValT* vals = (ValT*)(base + LY::vals);
    void* rec = base + LY::rec;
    uint32_t* keys = (uint32_t*)(base + LY::keys);
    uint32_t* stage = (uint32_t*)(base + LY::stage);
    const int r0 = bin_start[bin], r1 = bin_start[bin + 1];
    const int stride = gridDim.x * warps;
    int r = r0 + blockIdx.x * warps + warp;
    if (r >= r1) return;
    for (int t = lane; t < S; t += 32) {
        keys[t] = EMPTY;
        vals[t] = (ValT)0;
    }
    __syncwarp();
    // software pipeline over rows: the next row's bounds and first 32 A entries are
    // loaded during the current row's epilogue
    int i = perm[r];
    int64_t s = ld(arm, i), e = ld(arm, i + 1);
    int jn = 0;
    ValT an = (ValT)0;
    if (lane < e - s) {
        jn = __ldg(aent + s + lane);
        an = __ldg(aval + s + lane);
    }
    while (true) {
        const int64_t cb = ld(crm, i);
        const int clen = (int)(ld(crm, i + 1) - cb);
        const int rn = r + stride;
        const int inext = rn < r1 ? perm[rn] : -1;
        row_products<OffT, ValT, O32>(s, e, jn, an, aent, aval, brm, bent, bval, rec,
                                      [&](uint32_t col, ValT prod) {
                                     const bool act = col != EMPTY;
                                     const uint32_t h = strict_claim<S>(keys, col, act);
                                     if (act) vals[h] += prod;
                                 });
        if (dinv) {
            // Jacobi-fused row: scale E(i,:) by -omega D^-1(i), insert B(i,:)
            __syncwarp();
            const ValT sc = (ValT)(-omega * (double)__ldg(dinv + i));
            for (int t = lane; t < S; t += 32) vals[t] *= sc;
            __syncwarp();
            const int64_t bs = ld(brm, i), be = ld(brm, i + 1);
            for (int64_t q0 = bs; q0 < be; q0 += 32) {
                const bool act = q0 + lane < be;
                const uint32_t col = act ? (uint32_t)__ldg(bent + q0 + lane) : EMPTY;
                const uint32_t h = strict_claim<S>(keys, col, act);
                if (act) vals[h] += __ldg(bval + q0 + lane);
                __syncwarp();
            }
        }
        // next row's bounds (their loads overlap the epilogue)
        int64_t sn = 0, en = 0;
        if (inext >= 0) {
            sn = ld(arm, inext);
            en = ld(arm, inext + 1);
        }
        // ---- epilogue: compaction (slot order), sort, coalesced write, reset ----
        int n = 0;
        uint32_t mn = 0xffffffffu, mx = 0u;
#pragma unroll 4
        for (int c = 0; c < S / 32; ++c) {
            const uint32_t k = keys[c * 32 + lane];
            const bool occ = k != EMPTY;
            const unsigned bal = __ballot_sync(FULL, occ);
            if (occ) {
                const int pos = n + __popc(bal & lanemask_lt());
                if (pos < CAP) stage[pos] = (uint32_t)(c * 32 + lane);
                mn = min(mn, k);
                mx = max(mx, k);
            }
            n += __popc(bal);
        }
        __syncwarp();
        // next row's first A entries
        if (inext >= 0 && lane < en - sn) {
            jn = __ldg(aent + sn + lane);
            an = __ldg(aval + sn + lane);
        }
        const int nn = min(min(n, clen), CAP);  // guard: never write past the row
        if (SORT) {
            mn = __reduce_min_sync(FULL, mn);
            mx = __reduce_max_sync(FULL, mx);
            const bool packed = (mx - mn) < ((1u << (32 - LOGS)) - 1u);
            uint32_t v[E];
#pragma unroll
            for (int q = 0; q < E; ++q) {
                const int idx = lane * E + q;
                uint32_t w = 0xffffffffu;
                if (idx < nn) {
                    const uint32_t slot = stage[idx];
                    const uint32_t k = keys[slot];
                    w = packed ? (((k - mn) << LOGS) | slot) : k;
                }
                v[q] = w;
            }
            warp_bitonic_sort<E>(v);
            __syncwarp();
#pragma unroll
            for (int q = 0; q < E; ++q) {
                const int idx = lane * E + q;
                if (idx < nn) stage[idx] = v[q];
            }
            __syncwarp();
            for (int t = lane; t < nn; t += 32) {
                const uint32_t w = stage[t];
                uint32_t slot, col;
                if (packed) {
                    slot = w & (S - 1);
                    col = (w >> LOGS) + mn;
                } else {
                    col = w;
                    slot = strict_find<S>(keys, col);
                }
                cent[cb + t] = (int32_t)col;
                cval[cb + t] = vals[slot];
            }
        } else {
            for (int t = lane; t < nn; t += 32) {
                const uint32_t slot = stage[t];
                cent[cb + t] = (int32_t)keys[slot];
                cval[cb + t] = vals[slot];
            }
        }
        __syncwarp();
#pragma unroll 4
        for (int c = 0; c < S / 32; ++c) {
            keys[c * 32 + lane] = EMPTY;
            vals[c * 32 + lane] = (ValT)0;
        }
        __syncwarp();
        if (inext < 0) break;
        r = rn;
        i = inext;
        s = sn;
        e = en;
    }
}


// ------------------------------------------------------------------------------------
// a7 for rows whose pattern was kept by the symbolic phase (sorted (word, mask) pairs,
// <= 64 words).  The pattern fixes every column's position in the sorted output row:
// rank(c) = prefix(word(c)) + popc(mask & bits below c).  The words go into a small
// shared hash table (key = word, value = (mask, prefix)); each product looks its word up
// (the key is always present: no claims), computes its rank and accumulates into a
// dense per-row value array (accum = +).  The B row of a step has distinct
// columns (strictly sorted B), so ranks within a step are distinct and the update is a
// plain shared load/add/store.  Entries are written straight from the pattern and the
// values in order: the row is sorted without a sort.
// ------------------------------------------------------------------------------------
constexpr int PAT_W = 64;       // max words of a kept pattern (symbolic PAT_WORDS)
constexpr int PAT_NWIN = 2048;  // words of the widest symbolic window (64K bits)

constexpr int PAT_SW = 128;  // word-table slots (patterns whose words span > PAT_NWIN)

template <typename ValT, int CAP>
struct PatLayout {
    static constexpr size_t vals = 0;
    static constexpr size_t rec = ((size_t)CAP * sizeof(ValT) + 15) / 16 * 16;
    static constexpr size_t winfo = rec + REC_BYTES;
    static constexpr size_t wkeys = winfo + (size_t)PAT_SW * 8;
    static constexpr size_t widx = wkeys + (size_t)PAT_SW * 4;
    static constexpr size_t bytes = (widx + (size_t)PAT_NWIN + 15) / 16 * 16;
};

// word table of a pattern whose words are spread out: multiplicative hash, linear probing
__device__ __forceinline__ uint32_t wt_slot(uint32_t w) { return (w * 0x9E3779B1u) >> (32 - ilog2(PAT_SW)); }

// insert distinct words (write-then-verify claims); returns the slot
__device__ __forceinline__ uint32_t wt_insert(uint32_t* keys, uint32_t w, bool act) {
    uint32_t h = wt_slot(w);
    bool need = false;
    if (act) {
        while (keys[h] != EMPTY) h = (h + 1) & (PAT_SW - 1);
        need = true;
    }
    while (__any_sync(FULL, need)) {
        if (need) keys[h] = w;
        __syncwarp();
        if (need) {
            if (keys[h] == w) {
                need = false;
            } else {
                while (keys[h] != EMPTY) h = (h + 1) & (PAT_SW - 1);
            }
        }
        __syncwarp();
    }
    return h;
}

template <typename OffT, typename ValT, int CAP, bool O32, int MINB, bool DENSE>
__global__ void __launch_bounds__(256, MINB) k_num_pattern(const OffT* __restrict__ arm, const int32_t* __restrict__ aent,
                                                     const ValT* __restrict__ aval, const OffT* __restrict__ brm,
                                                     const int32_t* __restrict__ bent, const ValT* __restrict__ bval,
                                                     const OffT* __restrict__ crm, int32_t* __restrict__ cent,
                                                     ValT* __restrict__ cval, const int32_t* __restrict__ perm,
                                                     const int* __restrict__ bin_start, int bin,
                                                     const uint2* __restrict__ pat, const long long* __restrict__ pat_off,
                                                     const int* __restrict__ pat_len, const ValT* __restrict__ dinv,
                                                     double omega) {
    using LY = PatLayout<ValT, CAP>;
    extern __shared__ __align__(16) unsigned char sm_pat[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, warps = blockDim.x >> 5;
    unsigned char* base = sm_pat + (size_t)warp * LY::bytes;
    ValT* vals = (ValT*)(base + LY::vals);
    void* rec = base + LY::rec;
    uint32_t* wkeys = (uint32_t*)(base + LY::wkeys);
    const int r0 = bin_start[bin], r1 = bin_start[bin + 1];
    const int stride = gridDim.x * warps;
    int r = r0 + blockIdx.x * warps + warp;
    if (r >= r1) return;
    for (int t = lane; t < CAP; t += 32) vals[t] = (ValT)0;
    if (!DENSE)
        for (int t = lane; t < PAT_SW; t += 32) wkeys[t] = EMPTY;
    __syncwarp();
    int i = perm[r];
    int64_t s = ld(arm, i), e = ld(arm, i + 1);
    int jn = 0;
    ValT an = (ValT)0;
    if (lane < e - s) {
        jn = __ldg(aent + s + lane);
        an = __ldg(aval + s + lane);
    }
    while (true) {
        const int64_t cb = ld(crm, i);
        const int clen = (int)(ld(crm, i + 1) - cb);
        const long long po = pat_off[i];
        const int pl = pat_len[i];
        const int rn = r + stride;
        const int inext = rn < r1 ? perm[rn] : -1;
        // ---- the row's pattern: word table + entries ----
        const uint2 p0 = lane < pl ? pat[po + lane] : make_uint2(0u, 0u);
        const uint2 p1 = lane + 32 < pl ? pat[po + 32 + lane] : make_uint2(0u, 0u);
        const int c0 = __popc(p0.y), c1 = __popc(p1.y);
        int x0 = c0, x1 = c1;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const int y0 = __shfl_up_sync(FULL, x0, d), y1 = __shfl_up_sync(FULL, x1, d);
            if (lane >= d) {
                x0 += y0;
                x1 += y1;
            }
        }
        const int tot0 = __shfl_sync(FULL, x0, 31);
        const uint32_t pre0 = (uint32_t)(x0 - c0), pre1 = (uint32_t)(tot0 + x1 - c1);
        // word lookup: a dense index over the pattern's word span when it is narrow
        // (entries of other rows are never read), else a small hash table
        const uint32_t wb = __shfl_sync(FULL, p0.x, 0);
        const uint32_t wl_ = pl > 32 ? __shfl_sync(FULL, p1.x, (pl - 33) & 31) : __shfl_sync(FULL, p0.x, (pl - 1) & 31);
        (void)wl_;
        constexpr bool dense = DENSE;  // binning put the row here by its word span
        const uint32_t o_sw = (uint32_t)warp * (uint32_t)LY::bytes;
        uint32_t h0 = 0, h1 = 0;
        if constexpr (DENSE) {
            if (lane < pl) {
                sm_pat[o_sw + LY::widx + (p0.x - wb)] = (uint8_t)lane;
                *(uint2*)(sm_pat + o_sw + LY::winfo + lane * 8u) = make_uint2(p0.y, pre0);
            }
            if (lane + 32 < pl) {
                sm_pat[o_sw + LY::widx + (p1.x - wb)] = (uint8_t)(lane + 32);
                *(uint2*)(sm_pat + o_sw + LY::winfo + (lane + 32) * 8u) = make_uint2(p1.y, pre1);
            }
        } else {
            h0 = wt_insert(wkeys, p0.x, lane < pl);
            h1 = wt_insert(wkeys, p1.x, lane + 32 < pl);
            if (lane < pl) *(uint2*)(sm_pat + o_sw + LY::winfo + h0 * 8u) = make_uint2(p0.y, pre0);
            if (lane + 32 < pl) *(uint2*)(sm_pat + o_sw + LY::winfo + h1 * 8u) = make_uint2(p1.y, pre1);
        }
        {
            uint32_t m = p0.y;
            int o = (int)pre0;
            while (m) {
                const int b = __ffs(m) - 1;
                m &= m - 1;
                if (o < clen) cent[cb + o] = (int32_t)(p0.x * 32u + (uint32_t)b);
                ++o;
            }
            m = p1.y;
            o = (int)pre1;
            while (m) {
                const int b = __ffs(m) - 1;
                m &= m - 1;
                if (o < clen) cent[cb + o] = (int32_t)(p1.x * 32u + (uint32_t)b);
                ++o;
            }
        }
        __syncwarp();
        // ---- products: rank lookup + dense accumulate ----
        // (shared accesses go through sm_pat with 32-bit offsets: no generic addressing)
        const uint32_t o_idx = o_sw + (uint32_t)LY::widx - wb;
        const uint32_t o_inf = o_sw + (uint32_t)LY::winfo;
        const uint32_t o_val = o_sw + (uint32_t)LY::vals;
        auto mp_rank = [&](uint32_t wi, uint32_t col) {
            const uint2 mp = *(const uint2*)(sm_pat + o_inf + wi * 8u);
            return mp.y + __popc(mp.x & ((1u << (col & 31)) - 1u));
        };
        auto acc = [&](uint32_t rk, ValT prod) {
            if (rk < (uint32_t)CAP) *(ValT*)(sm_pat + o_val + rk * sizeof(ValT)) += prod;
        };
        if constexpr (DENSE) {
            row_products<OffT, ValT, O32>(s, e, jn, an, aent, aval, brm, bent, bval, rec,
                                          [&](uint32_t col, ValT prod) {
                                              if (col != EMPTY) acc(mp_rank(sm_pat[o_idx + (col >> 5)], col), prod);
                                              __syncwarp();
                                          });
        } else {
            row_products<OffT, ValT, O32>(s, e, jn, an, aent, aval, brm, bent, bval, rec,
                                          [&](uint32_t col, ValT prod) {
                                              if (col != EMPTY) {
                                                  const uint32_t w = col >> 5;
                                                  uint32_t wi = wt_slot(w);
                                                  while (wkeys[wi] != w) wi = (wi + 1) & (PAT_SW - 1);
                                                  acc(mp_rank(wi, col), prod);
                                              }
                                              __syncwarp();
                                          });
        }
        if (dinv) {
            // Jacobi-fused row: scale E(i,:) by -omega D^-1(i), add B(i,:)
            __syncwarp();
            const ValT sc = (ValT)(-omega * (double)__ldg(dinv + i));
            for (int t = lane; t < min(clen, CAP); t += 32) vals[t] *= sc;
            __syncwarp();
            const int64_t bs = ld(brm, i), be = ld(brm, i + 1);
            for (int64_t q0 = bs; q0 < be; q0 += 32) {
                if (q0 + lane < be) {
                    const uint32_t col = (uint32_t)__ldg(bent + q0 + lane);
                    const ValT bv = __ldg(bval + q0 + lane);
                    if constexpr (DENSE) {
                        acc(mp_rank(sm_pat[o_idx + (col >> 5)], col), bv);
                    } else {
                        const uint32_t w = col >> 5;
                        uint32_t wi = wt_slot(w);
                        while (wkeys[wi] != w) wi = (wi + 1) & (PAT_SW - 1);
                        acc(mp_rank(wi, col), bv);
                    }
                }
                __syncwarp();
            }
        }
        int64_t sn = 0, en = 0;
        if (inext >= 0) {
            sn = ld(arm, inext);
            en = ld(arm, inext + 1);
        }
        __syncwarp();
        // ---- write the values in order, reset ----
        const int nn = min(clen, CAP);
        for (int t = lane; t < nn; t += 32) {
            cval[cb + t] = vals[t];
            vals[t] = (ValT)0;
        }
        if constexpr (!DENSE) {
            if (lane < pl) wkeys[h0] = EMPTY;
            if (lane + 32 < pl) wkeys[h1] = EMPTY;
        }
        if (inext >= 0 && lane < en - sn) {
            jn = __ldg(aent + sn + lane);
            an = __ldg(aval + sn + lane);
        }
        __syncwarp();
        if (inext < 0) break;
        r = rn;
        i = inext;
        s = sn;
        e = en;
    }
}

// ------------------------------------------------------------------------------------
// a7 for pattern rows with a dense word index, lean form (k_num_rank).  The method is
// k_num_pattern's -- rank(c) = prefix(word(c)) + popc(mask & bits below c) from the
// pattern kept by symbolic, accum = + into a dense per-row value array (PAPER.md:178,
// Eq. 1) -- with the instruction stream cut down:
//   * each 32-entry A chunk becomes steps, one per 32-entry segment of its B rows (empty
//     B rows give none, a row of L entries ceil(L/32)), 16-byte records in windows of 32;
//   * steps are branch-free: lanes past the B row's end load a valid entry of it and
//     accumulate into a dump slot vals[CAP], so no divergent region per step;
//   * two steps per iteration, loads two steps ahead, and both steps' rank lookups are
//     issued before either read-modify-write (the lookups only read the pattern tables);
//   * the prologue writes each rank's column into shared memory once (one popcount scan
//     of two 16-bit halves), and the epilogue writes entries and values coalesced.
// Needs B.nnz < 2^31 (32-bit element offsets) and strictly increasing B rows.  HASHW: the
// word index is a hash of the pattern's words (rows whose words span > PAT_NWIN words).
// ------------------------------------------------------------------------------------
// HASHW: patterns whose words span more than PAT_NWIN words (wide rows, e.g. C5): the word
// index is a PAT_SW-slot hash of the words (winfo indexed by hash slot) instead of a dense
// u8 index over the window.
template <typename ValT, int CAP, bool HASHW = false>
struct RankLayout {
    static constexpr size_t vals = 0;  // CAP + 1 values (slot CAP: idle lanes)
    static constexpr size_t cols = ((size_t)(CAP + 1) * sizeof(ValT) + 15) / 16 * 16;  // CAP int32
    static constexpr size_t rec = cols + (size_t)CAP * 4;                                // 32 x {bb, len, a}
    static constexpr size_t winfo = rec + 32 * 16;                  // (mask, prefix) per word / hash slot
    static constexpr size_t widx = winfo + (size_t)(HASHW ? PAT_SW : PAT_W) * 8;  // u8 index | hash keys
    static constexpr size_t bytes = (widx + (HASHW ? (size_t)PAT_SW * 4 : (size_t)PAT_NWIN) + 15) / 16 * 16;
};

template <typename OffT, typename ValT, int CAP, int MINB, bool HASHW>
__global__ void __launch_bounds__(256, MINB) k_num_rank(const OffT* __restrict__ arm, const int32_t* __restrict__ aent,
                                                        const ValT* __restrict__ aval, const OffT* __restrict__ brm,
                                                        const int32_t* __restrict__ bent, const ValT* __restrict__ bval,
                                                        const OffT* __restrict__ crm, int32_t* __restrict__ cent,
                                                        ValT* __restrict__ cval, const int32_t* __restrict__ perm,
                                                        const int* __restrict__ bin_start, int bin,
                                                        const uint2* __restrict__ pat, const long long* __restrict__ pat_off,
                                                        const int* __restrict__ pat_len, const ValT* __restrict__ dinv,
                                                        double omega) {
    using LY = RankLayout<ValT, CAP, HASHW>;
    extern __shared__ __align__(16) unsigned char sm_rank[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, warps = blockDim.x >> 5;
    // all shared accesses as sm_rank + 32-bit offset (shared addressing, no generic)
    const uint32_t o_w = (uint32_t)warp * (uint32_t)LY::bytes;
    const uint32_t o_val = o_w + (uint32_t)LY::vals, o_col = o_w + (uint32_t)LY::cols;
    const uint32_t o_rec = o_w + (uint32_t)LY::rec, o_inf = o_w + (uint32_t)LY::winfo;
    const int r0 = bin_start[bin], r1 = bin_start[bin + 1];
    const int stride = gridDim.x * warps;
    int r = r0 + blockIdx.x * warps + warp;
    if (r >= r1) return;
    for (int t = lane; t < CAP; t += 32) *(ValT*)(sm_rank + o_val + t * (uint32_t)sizeof(ValT)) = (ValT)0;
    uint32_t* wkeys = (uint32_t*)(sm_rank + o_w + (uint32_t)LY::widx);  // HASHW only
    if (HASHW)
        for (int t = lane; t < PAT_SW; t += 32) wkeys[t] = EMPTY;
    int i = perm[r];
    while (true) {
        const int rn = r + stride;
        const int inext = rn < r1 ? __ldg(perm + rn) : -1;
        const int64_t s = ld(arm, i), e = ld(arm, i + 1);
        const int64_t cb = ld(crm, i);
        const int clen = (int)(ld(crm, i + 1) - cb);
        const long long po = __ldg(pat_off + i);
        const int pl = __ldg(pat_len + i);
        // ---- the row's pattern: (mask, prefix) per word, word index, column of each rank ----
        const uint2 p0 = lane < pl ? __ldg(pat + po + lane) : make_uint2(0u, 0u);
        uint2 p1 = make_uint2(0u, 0u);
        if (pl > 32 && lane + 32 < pl) p1 = __ldg(pat + po + 32 + lane);
        const int c0 = __popc(p0.y), c1 = __popc(p1.y);
        int x = c0 | (c1 << 16);  // both halves' counts at once (each total <= 2048)
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const int y = __shfl_up_sync(FULL, x, d);
            if (lane >= d) x += y;
        }
        const int tot = __shfl_sync(FULL, x, 31);
        const int pre0 = (x & 0xffff) - c0;
        const int pre1 = (tot & 0xffff) + (x >> 16) - c1;
        const uint32_t wb = __shfl_sync(FULL, p0.x, 0);
        const uint32_t o_idx = o_w + (uint32_t)LY::widx - wb;
        __syncwarp();
        // word -> (mask, prefix) slot: dense u8 index, or the hash slot of the word
        uint32_t h0 = (uint32_t)lane, h1 = (uint32_t)lane + 32u;
        if constexpr (HASHW) {
            h0 = wt_insert(wkeys, p0.x, lane < pl);
            h1 = wt_insert(wkeys, p1.x, lane + 32 < pl);
        }
        if (lane < pl) {
            if constexpr (!HASHW) sm_rank[o_idx + p0.x] = (uint8_t)lane;
            *(uint2*)(sm_rank + o_inf + h0 * 8u) = make_uint2(p0.y, (uint32_t)pre0);
            uint32_t m = p0.y;
            uint32_t o = o_col + (uint32_t)pre0 * 4u;
            while (m) {
                *(int32_t*)(sm_rank + o) = (int32_t)(p0.x * 32u + (uint32_t)(__ffs(m) - 1));
                m &= m - 1;
                o += 4;
            }
        }
        if (lane + 32 < pl) {
            if constexpr (!HASHW) sm_rank[o_idx + p1.x] = (uint8_t)(lane + 32);
            *(uint2*)(sm_rank + o_inf + h1 * 8u) = make_uint2(p1.y, (uint32_t)pre1);
            uint32_t m = p1.y;
            uint32_t o = o_col + (uint32_t)pre1 * 4u;
            while (m) {
                *(int32_t*)(sm_rank + o) = (int32_t)(p1.x * 32u + (uint32_t)(__ffs(m) - 1));
                m &= m - 1;
                o += 4;
            }
        }
        __syncwarp();
        auto rank = [&](int col, bool valid) -> uint32_t {
            uint32_t wi;
            if constexpr (HASHW) {
                const uint32_t w = (uint32_t)col >> 5;
                wi = wt_slot(w);
                while (wkeys[wi] != w) wi = (wi + 1) & (PAT_SW - 1);  // present: no empty-slot test
            } else {
                wi = sm_rank[o_idx + ((uint32_t)col >> 5)];
            }
            const uint2 mp = *(const uint2*)(sm_rank + o_inf + wi * 8u);
            const uint32_t rk = mp.y + __popc(mp.x & ~(0xffffffffu << (col & 31)));
            return valid ? rk : (uint32_t)CAP;
        };
        auto acc = [&](uint32_t rk, ValT prod) {
            ValT* p = (ValT*)(sm_rank + o_val + rk * (uint32_t)sizeof(ValT));
            *p += prod;
        };
        // ---- products, one 32-entry A chunk at a time ----
        // A step is one 32-entry segment of a B row (a B row of L entries gives ceil(L/32)
        // steps); the chunk's steps are written as 16-byte records in windows of 32.
        for (int64_t a0 = s; a0 < e; a0 += 32) {
            const int na = (int)min((int64_t)32, e - a0);
            int bb = 0, bl = 0;
            double av = 0.0;
            if (lane < na) {
                const int j = __ldg(aent + a0 + lane);
                av = (double)__ldg(aval + a0 + lane);
                bb = (int)ld(brm, j);
                bl = (int)(ld(brm, j + 1) - bb);
            }
            // the chunk's nt steps from their records: two per iteration, loads two ahead
            auto run_steps = [&](int nt) {
                auto load = [&](int t, int& col, ValT& bv, ValT& a, bool& valid) {
                    const int4 rr = *(const int4*)(sm_rank + o_rec + (uint32_t)min(t, nt - 1) * 16u);
                    valid = t < nt && lane < rr.y;
                    const int q = rr.x + min(lane, rr.y - 1);
                    col = __ldg(bent + q);
                    bv = __ldg(bval + q);
                    a = (ValT)__hiloint2double(rr.w, rr.z);
                };
                int colA, colB;
                ValT bA, bB, aA, aB;
                bool vA, vB;
                load(0, colA, bA, aA, vA);
                load(1, colB, bB, aB, vB);
                for (int t = 0; t < nt; t += 2) {
                    const uint32_t rA = rank(colA, vA), rB = rank(colB, vB);
                    const ValT pA = aA * bA, pB = aB * bB;
                    if (t + 2 < nt) {
                        load(t + 2, colA, bA, aA, vA);
                        load(t + 3, colB, bB, aB, vB);
                    }
                    acc(rA, pA);
                    __syncwarp();
                    acc(rB, pB);
                    __syncwarp();
                }
            };
            // (HASHW rows -- wide patterns, e.g. C5's 81-entry B rows -- always take the
            // segment form: one call site of run_steps measured 221 vs 325 ms on C5)
            const int maxbl = HASHW ? 33 : (int)__reduce_max_sync(FULL, (unsigned)bl);
            if (maxbl <= 32) {
                // one step per non-empty B row: records compacted by ballot
                const unsigned ne = __ballot_sync(FULL, bl > 0);
                __syncwarp();
                if (bl > 0)
                    *(int4*)(sm_rank + o_rec + __popc(ne & lanemask_lt()) * 16u) =
                        make_int4(bb, bl, __double2loint(av), __double2hiint(av));
                __syncwarp();
                if (ne) run_steps(__popc(ne));
            } else {
                // long B rows: one step per 32-entry segment, records in windows of 32
                const int nseg = (bl + 31) >> 5;
                int xs = nseg;
#pragma unroll
                for (int d = 1; d < 32; d <<= 1) {
                    const int y = __shfl_up_sync(FULL, xs, d);
                    if (lane >= d) xs += y;
                }
                const int T = __shfl_sync(FULL, xs, 31);
                const int ex = xs - nseg;
                for (int w0 = 0; w0 < T; w0 += 32) {
                    __syncwarp();
                    for (int g = max(ex, w0); g < min(ex + nseg, w0 + 32); ++g) {
                        const int so = (g - ex) * 32;
                        *(int4*)(sm_rank + o_rec + (uint32_t)(g - w0) * 16u) =
                            make_int4(bb + so, min(32, bl - so), __double2loint(av), __double2hiint(av));
                    }
                    __syncwarp();
                    run_steps(min(32, T - w0));
                }
            }
            __syncwarp();
        }
        if (dinv) {
            // Jacobi-fused row: C(i,:) = B(i,:) - omega D^-1(i) E(i,:).
            // E(i,:) is scaled once per entry by the row's scalar, then B(i,:) is added at
            // its ranks (its columns lie in E's pattern when A(i,i) is stored).
            const ValT sc = (ValT)(-omega * (double)__ldg(dinv + i));
            for (int t = lane; t < clen; t += 32) *(ValT*)(sm_rank + o_val + (uint32_t)t * (uint32_t)sizeof(ValT)) *= sc;
            __syncwarp();
            const int bs = (int)ld(brm, i), bl = (int)(ld(brm, i + 1) - bs);
            for (int q0 = 0; q0 < bl; q0 += 32) {
                const bool valid = q0 + lane < bl;
                const int q = bs + min(q0 + lane, bl - 1);
                const int col = __ldg(bent + q);
                // a word outside the dense index's range is not in the pattern
                bool inpat = HASHW || ((uint32_t)col >> 5) - wb < (uint32_t)PAT_NWIN;
                if constexpr (HASHW) {
                    // the word must be present before probing (no empty-slot test in rank())
                    const uint32_t w = (uint32_t)col >> 5;
                    uint32_t wi = wt_slot(w);
                    while (wkeys[wi] != w && wkeys[wi] != EMPTY) wi = (wi + 1) & (PAT_SW - 1);
                    inpat = wkeys[wi] == w;
                }
                uint32_t rk = rank(inpat ? col : (int)(wb * 32u), valid && inpat);
                // a column outside the pattern (A(i,i) not stored) must not land on another rank
                if (rk < (uint32_t)CAP && *(const int32_t*)(sm_rank + o_col + rk * 4u) != col) rk = CAP;
                acc(rk, __ldg(bval + q));
                __syncwarp();
            }
        }
        // ---- entries and values, coalesced; reset ----
        if (HASHW) {
            if (lane < pl) wkeys[h0] = EMPTY;
            if (lane + 32 < pl) wkeys[h1] = EMPTY;
        }
        for (int t = lane; t < clen; t += 32) {
            // C is written once and not read again here: streaming (evict-first) stores keep
            // L2 for B's rows, which neighbouring rows of C read again
            __stcs(cent + cb + t, *(const int32_t*)(sm_rank + o_col + (uint32_t)t * 4u));
            ValT* p = (ValT*)(sm_rank + o_val + (uint32_t)t * (uint32_t)sizeof(ValT));
            __stcs(cval + cb + t, *p);
            *p = (ValT)0;
        }
        __syncwarp();
        if (inext < 0) break;
        r = rn;
        i = inext;
    }
}

// KK_NUM_RANK=0 selects k_num_pattern for the dense-index pattern bins (experiments)
static bool use_num_rank() {
    static const bool v = [] {
        const char* s = getenv("KK_NUM_RANK");
        return !(s && s[0] == '0');
    }();
    return v;
}

template <typename OffT, typename ValT, int CAP, bool HASHW = false>
static void launch_num_rank(Launch& L, const NumArgs& a, int bin) {
    const int rows = a.host_bin_start[bin + 1] - a.host_bin_start[bin];
    if (rows <= 0) return;
    const int warps = 8;
    const size_t smem = (size_t)warps * RankLayout<ValT, CAP, HASHW>::bytes;
    static const int minb = [] {
        const char* v = getenv("KK_RANK_MINB");
        const int x = v ? atoi(v) : 4;
        return (x == 5 || x == 6) ? x : 4;
    }();
    auto kern = minb == 5 ? k_num_rank<OffT, ValT, CAP, 5, HASHW>
              : minb == 6 ? k_num_rank<OffT, ValT, CAP, 6, HASHW>
                          : k_num_rank<OffT, ValT, CAP, 4, HASHW>;
    KCfg c = kernel_cfg(kern, warps * 32, smem, L.num_sms);
    int64_t need = (rows + warps - 1) / warps;
    int grid = (int)std::min<int64_t>(need, c.grid_cap);
    L.begin(kname(HASHW ? "num_rank_hash" : "num_rank", CAP), L.stream);
    kern<<<grid, warps * 32, smem, L.stream>>>((const OffT*)a.A.row_map, a.A.entries, (const ValT*)a.A.values,
                                               (const OffT*)a.B.row_map, a.B.entries, (const ValT*)a.B.values,
                                               (const OffT*)a.c_row_map, a.c_entries, (ValT*)a.c_values, a.perm,
                                               a.bin_start, bin, a.pat, a.pat_off, a.pat_len, (const ValT*)a.dinv, a.omega);
    L.end(L.stream);
}

template <typename OffT, typename ValT, int CAP, bool DENSE>
static void launch_num_pattern(Launch& L, const NumArgs& a, int bin) {
    if (a.B.nnz < INT32_MAX && use_num_rank()) {
        launch_num_rank<OffT, ValT, CAP, !DENSE>(L, a, bin);
        return;
    }
    const int rows = a.host_bin_start[bin + 1] - a.host_bin_start[bin];
    if (rows <= 0) return;
    const int warps = 8;
    const size_t smem = (size_t)warps * PatLayout<ValT, CAP>::bytes;
    // resident CTAs per SM the register budget targets: 4 (60 registers, no spills) measured
    // fastest on C2; KK_PAT_MINB=5|6 for experiments
    static const int minb = [] {
        const char* v = getenv("KK_PAT_MINB");
        const int x = v ? atoi(v) : 4;
        return (x == 5 || x == 6) ? x : 4;
    }();
    auto kern = a.B.nnz >= INT32_MAX ? k_num_pattern<OffT, ValT, CAP, false, 4, DENSE>
              : minb == 5            ? k_num_pattern<OffT, ValT, CAP, true, 5, DENSE>
              : minb == 6            ? k_num_pattern<OffT, ValT, CAP, true, 6, DENSE>
                                     : k_num_pattern<OffT, ValT, CAP, true, 4, DENSE>;
    KCfg c = kernel_cfg(kern, warps * 32, smem, L.num_sms);
    int64_t need = (rows + warps - 1) / warps;
    int grid = (int)std::min<int64_t>(need, c.grid_cap);
    L.begin(kname(DENSE ? "num_pattern" : "num_pattern_hash", CAP), L.stream);
    kern<<<grid, warps * 32, smem, L.stream>>>((const OffT*)a.A.row_map, a.A.entries, (const ValT*)a.A.values,
                                               (const OffT*)a.B.row_map, a.B.entries, (const ValT*)a.B.values,
                                               (const OffT*)a.c_row_map, a.c_entries, (ValT*)a.c_values, a.perm,
                                               a.bin_start, bin, a.pat, a.pat_off, a.pat_len, (const ValT*)a.dinv, a.omega);
    L.end(L.stream);
}

// rows of numeric bin `bin` hold nnz(C_i) <= CAP = 16 << bin; the table has S = 4*CAP slots
template <typename OffT, typename ValT, int CAP, int F, bool SORT>
static void launch_num_strict_f(Launch& L, const NumArgs& a, int bin) {
    constexpr int S = F * CAP;
    const int rows = a.host_bin_start[bin + 1] - a.host_bin_start[bin];
    if (rows <= 0) return;
    const int warps = CAP <= 128 ? 8 : 4;
    const size_t smem = (size_t)warps * StrictLayout<ValT, S, CAP>::bytes;
    auto kern = a.B.nnz < INT32_MAX ? k_num_strict<OffT, ValT, S, CAP, SORT, true>
                                    : k_num_strict<OffT, ValT, S, CAP, SORT, false>;
    KCfg c = kernel_cfg(kern, warps * 32, smem, L.num_sms);
    int64_t need = (rows + warps - 1) / warps;
    int grid = (int)std::min<int64_t>(need, c.grid_cap);
    L.begin(kname("num_strict", S), L.stream);
    kern<<<grid, warps * 32, smem, L.stream>>>((const OffT*)a.A.row_map, a.A.entries, (const ValT*)a.A.values,
                                               (const OffT*)a.B.row_map, a.B.entries, (const ValT*)a.B.values,
                                               (const OffT*)a.c_row_map, a.c_entries, (ValT*)a.c_values, a.perm,
                                               a.bin_start, bin, (const ValT*)a.dinv, a.omega);
    L.end(L.stream);
}

// table factor S / CAP (load factor <= 1/F).  F = 2 measured faster than 4 on C2 (smaller
// tables -> more resident warps); KK_NUM_TABLE_FACTOR=4 selects 4 (experiments).
static int num_table_factor() {
    static int f = [] {
        const char* v = getenv("KK_NUM_TABLE_FACTOR");
        return (v && atoi(v) == 4) ? 4 : 2;
    }();
    return f;
}

template <typename OffT, typename ValT, int CAP, bool SORT>
static void launch_num_strict(Launch& L, const NumArgs& a, int bin) {
    if (num_table_factor() == 4)
        launch_num_strict_f<OffT, ValT, CAP, 4, SORT>(L, a, bin);
    else
        launch_num_strict_f<OffT, ValT, CAP, 2, SORT>(L, a, bin);
}


// ------------------------------------------------------------------------------------
// a7 for long rows (nnz(C_i) > 512) when B has at most ~1.4M columns: a CTA owns a row and
// the row's whole column bit vector (k bits) plus the popcount prefix of every group of 4
// words in shared memory.  (1) the bit vector of the row's pattern (accum = OR, as the
// symbolic dense tier); (2) one pass over it writes the sorted column indices of C(i,:)
// and the group prefixes; (3) each product finds its rank in the row (group prefix +
// popcounts of <= 3 preceding words + the bits below it) and is added to C's value at that
// position in global memory (fp64/fp32 reduction at L2, fire-and-forget).  This is the
// paper's dense accumulator turned into "bit vector in shared memory,
// scalar array = the output row itself", so no column windows are walked.
// ------------------------------------------------------------------------------------
constexpr int HUB_THREADS = 512;
constexpr int HUB_WARPS = HUB_THREADS / 32;

__host__ __device__ constexpr int64_t hub_words(int64_t k) { return ((k + 127) / 128) * 4; }  // multiple of 4
constexpr int HUB_LONG = 256;     // B rows longer than this are walked by the whole CTA
constexpr int HUB_LIST = 1024;    // capacity of the per-row list of such A entries

// shared layout: bm[NW] | gp[NW/4] (padded to 8 bytes) | wtot[HUB_WARPS] (int64) |
//                list[HUB_LIST] (int32) | nlist
__host__ __device__ constexpr int64_t hub_gp_words(int64_t k) { return (hub_words(k) / 4 + 1) & ~1ll; }
__host__ __device__ constexpr size_t hub_smem(int64_t k) {
    return (size_t)(hub_words(k) + hub_gp_words(k)) * 4 + (size_t)HUB_WARPS * 8 + (size_t)HUB_LIST * 4 + 16;
}

template <typename OffT, typename ValT>
__global__ void __launch_bounds__(HUB_THREADS, 1) k_num_hub(const OffT* __restrict__ arm, const int32_t* __restrict__ aent,
                                                             const ValT* __restrict__ aval, const OffT* __restrict__ brm,
                                                             const int32_t* __restrict__ bent, const ValT* __restrict__ bval,
                                                             const OffT* __restrict__ crm, int32_t* __restrict__ cent,
                                                             ValT* __restrict__ cval, const int32_t* __restrict__ perm,
                                                             const int* __restrict__ bin_start, int bin, int64_t k) {
    extern __shared__ __align__(16) uint32_t sm_hub[];
    const int64_t NW = hub_words(k);
    uint32_t* bm = sm_hub;
    uint32_t* gp = bm + NW;
    long long* wtot = (long long*)(gp + hub_gp_words(k));
    int* list = (int*)(wtot + HUB_WARPS);
    int* nlist = list + HUB_LIST;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int r0 = bin_start[bin], r1 = bin_start[bin + 1];
    if (r0 + (int)blockIdx.x >= r1) return;
    const int64_t per = (NW / 4 + HUB_WARPS - 1) / HUB_WARPS * 4;  // words per warp (multiple of 4)
    for (int r = r0 + blockIdx.x; r < r1; r += gridDim.x) {
        const int i = perm[r];
        const int64_t s = ld(arm, i), e = ld(arm, i + 1);
        const int64_t cb = ld(crm, i);
        const int64_t clen = ld(crm, i + 1) - cb;
        for (int64_t t = threadIdx.x; t < NW / 4; t += HUB_THREADS) ((uint4*)bm)[t] = make_uint4(0, 0, 0, 0);
        if (threadIdx.x == 0) *nlist = 0;
        __syncthreads();
        // (1) pattern.  Warps take the A entries whose B rows are short; longer B rows are
        // listed and then walked by the whole CTA, one at a time (a hub B row must not
        // leave one warp working while the others wait at the barrier).
        for (int64_t p = s + warp; p < e; p += HUB_WARPS) {
            const int j = __ldg(aent + p);
            const int64_t bs = ld(brm, j), be = ld(brm, j + 1);
            if (be - bs > HUB_LONG) {
                int slot = 0;
                if (lane == 0) slot = atomicAdd(nlist, 1);
                slot = __shfl_sync(FULL, slot, 0);
                if (slot < HUB_LIST) {
                    if (lane == 0) list[slot] = (int)(p - s);
                    continue;
                }
            }
            for (int64_t q = bs + lane; q < be; q += 32) {
                const int c = __ldg(bent + q);
                atomicOr(&bm[c >> 5], 1u << (c & 31));
            }
        }
        __syncthreads();
        const int nl = min(*nlist, HUB_LIST);
        for (int l = 0; l < nl; ++l) {
            const int j = __ldg(aent + s + list[l]);
            const int64_t bs = ld(brm, j), be = ld(brm, j + 1);
            for (int64_t q = bs + threadIdx.x; q < be; q += HUB_THREADS) {
                const int c = __ldg(bent + q);
                atomicOr(&bm[c >> 5], 1u << (c & 31));
            }
        }
        __syncthreads();
        // (2) per-warp word ranges: totals, then prefixes + sorted entries in one pass
        const int64_t w0 = (int64_t)warp * per, w1 = min(NW, w0 + per);
        long long tot = 0;
        for (int64_t w = w0 + lane; w < w1; w += 32) tot += __popc(bm[w]);
        tot = warp_sum(tot);
        if (lane == 0) wtot[warp] = tot;
        __syncthreads();
        long long base = 0;
        for (int w = 0; w < warp; ++w) base += wtot[w];
        for (int64_t c0 = w0; c0 < w1; c0 += 32) {
            const int64_t w = c0 + lane;
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
                if (pos < clen) cent[cb + pos] = (int32_t)(w * 32 + b);
                ++pos;
            }
            base += __shfl_sync(FULL, x, 31);
        }
        for (int64_t t = threadIdx.x; t < clen; t += HUB_THREADS) cval[cb + t] = (ValT)0;
        __syncthreads();
        // (3) values: rank lookup, reduction into C(i, rank) (same split of the work)
        auto add = [&](int c, ValT prod) {
            const int w = c >> 5;
            uint32_t rk = gp[w >> 2];
            const int g0 = w & ~3;
            if (g0 + 0 < w) rk += __popc(bm[g0 + 0]);
            if (g0 + 1 < w) rk += __popc(bm[g0 + 1]);
            if (g0 + 2 < w) rk += __popc(bm[g0 + 2]);
            rk += __popc(bm[w] & ((1u << (c & 31)) - 1u));
            if ((int64_t)rk < clen) atomicAdd(&cval[cb + rk], prod);
        };
        for (int64_t p = s + warp; p < e; p += HUB_WARPS) {
            const int j = __ldg(aent + p);
            const int64_t bs = ld(brm, j), be = ld(brm, j + 1);
            if (be - bs > HUB_LONG && nl > 0) {
                // listed above (unless the list overflowed: then it is not in the list)
                bool listed = false;
                for (int l = lane; l < nl; l += 32) listed |= list[l] == (int)(p - s);
                if (__any_sync(FULL, listed)) continue;
            }
            const ValT a = __ldg(aval + p);
            for (int64_t q = bs + lane; q < be; q += 32) add(__ldg(bent + q), a * __ldg(bval + q));
        }
        for (int l = 0; l < nl; ++l) {
            const int64_t p = s + list[l];
            const int j = __ldg(aent + p);
            const ValT a = __ldg(aval + p);
            const int64_t bs = ld(brm, j), be = ld(brm, j + 1);
            for (int64_t q = bs + threadIdx.x; q < be; q += HUB_THREADS) add(__ldg(bent + q), a * __ldg(bval + q));
        }
        __syncthreads();
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
                                               a.bin_start, bin, a.logG, a.st, (const ValT*)a.dinv, a.omega);
    L.end(L.stream);
}

// a7 + a8 for tiny rows (flops_i <= TINY_MAX): a lane owns a row; columns and values in a
// register list (TinyList, accum = +), sorted by a transposition network and
// written to the row.  Jacobi-fused: E(i,:) scaled by -omega D^-1(i),
// then B(i,:) inserted.
template <typename OffT, typename ValT>
__global__ void __launch_bounds__(256) k_num_tiny(const OffT* __restrict__ arm, const int32_t* __restrict__ aent,
                                                  const ValT* __restrict__ aval, const OffT* __restrict__ brm,
                                                  const int32_t* __restrict__ bent, const ValT* __restrict__ bval,
                                                  const OffT* __restrict__ crm, int32_t* __restrict__ cent,
                                                  ValT* __restrict__ cval, const int32_t* __restrict__ perm,
                                                  const int* __restrict__ bin_start, int bin,
                                                  const ValT* __restrict__ dinv, double omega) {
    const int r0 = bin_start[bin], r1 = bin_start[bin + 1];
    for (int r = r0 + blockIdx.x * blockDim.x + threadIdx.x; r < r1; r += gridDim.x * blockDim.x) {
        const int i = perm[r];
        TinyList<TINY_MAX, ValT, true> T;
        const int64_t s = ld(arm, i), e = ld(arm, i + 1);
        for (int64_t p = s; p < e; ++p) {
            const int j = __ldg(aent + p);
            const ValT a = __ldg(aval + p);
            const int64_t bs = ld(brm, j), be = ld(brm, j + 1);
            for (int64_t q = bs; q < be; ++q) T.insert(__ldg(bent + q), a * __ldg(bval + q));
        }
        if (dinv) {
            T.scale((ValT)(-omega * (double)__ldg(dinv + i)));
            const int64_t bs = ld(brm, i), be = ld(brm, i + 1);
            for (int64_t q = bs; q < be; ++q) T.insert(__ldg(bent + q), __ldg(bval + q));
        }
        T.sort();
        const int64_t cb = ld(crm, i);
        const int clen = (int)(ld(crm, i + 1) - cb);
        const int nn = min(T.n, clen);
#pragma unroll
        for (int k = 0; k < TINY_MAX; ++k) {
            if (k < nn) {
                cent[cb + k] = T.cols[k];
                cval[cb + k] = T.vals[k];
            }
        }
    }
}

template <typename OffT, typename ValT>
static void launch_num_tiny(Launch& L, const NumArgs& a) {
    const int rows = a.host_bin_start[NUM_TINY_BIN + 1] - a.host_bin_start[NUM_TINY_BIN];
    if (rows <= 0) return;
    auto kern = k_num_tiny<OffT, ValT>;
    KCfg c = kernel_cfg(kern, 256, 0, L.num_sms);
    const int grid = (int)std::min<int64_t>((rows + 255) / 256, c.grid_cap);
    L.begin("num_tiny", L.stream);
    kern<<<grid, 256, 0, L.stream>>>((const OffT*)a.A.row_map, a.A.entries, (const ValT*)a.A.values,
                                     (const OffT*)a.B.row_map, a.B.entries, (const ValT*)a.B.values,
                                     (const OffT*)a.c_row_map, a.c_entries, (ValT*)a.c_values, a.perm, a.bin_start,
                                     NUM_TINY_BIN, (const ValT*)a.dinv, a.omega);
    L.end(L.stream);
}

template <typename OffT, typename ValT, bool SORT>
static void numeric_bins_t(Launch& L, const NumArgs& a, cudaStream_t dense_stream) {
    const int drows = a.host_bin_start[NUM_DENSE_BIN + 1] - a.host_bin_start[NUM_DENSE_BIN];
    const size_t hsm = hub_smem(a.k);
    static const bool force_windowed = [] {  // KK_NUM_WINDOWED=1: windowed dense tier for all k
        const char* v = getenv("KK_NUM_WINDOWED");
        return v && v[0] == '1';
    }();
    if (drows > 0 && a.k > 25600 && hsm <= 220 * 1024 && !force_windowed) {
        // long rows, one column window would not do: bit vector over all of k (k_num_hub)
        auto kern = k_num_hub<OffT, ValT>;
        KCfg c = kernel_cfg(kern, HUB_THREADS, hsm, L.num_sms);
        const int grid = (int)std::min<int64_t>(drows, c.grid_cap);
        cudaStream_t s = dense_stream ? dense_stream : L.stream;
        L.begin("num_hub", s);
        kern<<<grid, HUB_THREADS, hsm, s>>>((const OffT*)a.A.row_map, a.A.entries, (const ValT*)a.A.values,
                                            (const OffT*)a.B.row_map, a.B.entries, (const ValT*)a.B.values,
                                            (const OffT*)a.c_row_map, a.c_entries, (ValT*)a.c_values, a.perm,
                                            a.bin_start, NUM_DENSE_BIN, a.k);
        L.end(s);
    } else if (drows > 0) {
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
    launch_num_tiny<OffT, ValT>(L, a);
    if (a.pat) {
        launch_num_pattern<OffT, ValT, 512, true>(L, a, NUM_PAT_BIN0 + 4);
        launch_num_pattern<OffT, ValT, 256, true>(L, a, NUM_PAT_BIN0 + 3);
        launch_num_pattern<OffT, ValT, 128, true>(L, a, NUM_PAT_BIN0 + 2);
        launch_num_pattern<OffT, ValT, 64, true>(L, a, NUM_PAT_BIN0 + 1);
        launch_num_pattern<OffT, ValT, 32, true>(L, a, NUM_PAT_BIN0);
        launch_num_pattern<OffT, ValT, 512, false>(L, a, NUM_PATH_BIN0 + 3);
        launch_num_pattern<OffT, ValT, 256, false>(L, a, NUM_PATH_BIN0 + 2);
        launch_num_pattern<OffT, ValT, 128, false>(L, a, NUM_PATH_BIN0 + 1);
        launch_num_pattern<OffT, ValT, 64, false>(L, a, NUM_PATH_BIN0);
    }
    if (a.strict && a.logG >= 4) {
        launch_num_strict<OffT, ValT, 512, SORT>(L, a, 5);
        launch_num_strict<OffT, ValT, 256, SORT>(L, a, 4);
        launch_num_strict<OffT, ValT, 128, SORT>(L, a, 3);
        launch_num_strict<OffT, ValT, 64, SORT>(L, a, 2);
        launch_num_strict<OffT, ValT, 32, SORT>(L, a, 1);
    } else {
        launch_num_warp<OffT, ValT, 1024, SORT>(L, a, 5);
        launch_num_warp<OffT, ValT, 512, SORT>(L, a, 4);
        launch_num_warp<OffT, ValT, 256, SORT>(L, a, 3);
        launch_num_warp<OffT, ValT, 128, SORT>(L, a, 2);
        launch_num_warp<OffT, ValT, 64, SORT>(L, a, 1);
    }
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

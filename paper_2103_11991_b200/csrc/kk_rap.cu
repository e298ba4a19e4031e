// kk_rap.cu -- NEXT-4: fused single-pass Galerkin triple product Ac = R * A * P (the
// multigrid use of SpGEMM the paper motivates), two phases like the
// plain product: symbolic counts the distinct columns of every coarse
// row, numeric accumulates
//     Ac(I, c) = sum_{i in R(I,:)} r_Ii * sum_{j in A(i,:)} a_ij * P(j, c)        (Eq. 1 twice)
// without forming T = A*P.  A warp owns a coarse row I: its R entries are taken 4 per warp
// step (8 lanes each walk A(i,:) of one of them, longer A rows in rounds of 8), every lane
// walks the P rows of its A entries, and each product r*a*p is inserted into a warp-owned
// shared hash table keyed by column (accum = +).  The numeric epilogue sorts
// the row by a warp bitonic sort of packed (column - min) << log2 S | slot keys (as the
// hash tiers of the plain product).  Rows with more than RAP_CAP distinct columns are
// reported and the call fails (the two-product path handles them).
#include "kk_device.cuh"

#include <type_traits>

namespace kk {

constexpr int RAP_S = 512;    // table slots per warp
constexpr int RAP_CAP = 256;  // distinct columns of a coarse row (load factor <= 1/2)
constexpr int RAP_WARPS = 4;

// probe_claim with at most S probes: returns S when the table is full (symbolic flags the row)
template <int S>
__device__ __forceinline__ uint32_t rap_claim(uint32_t* keys, uint32_t key, bool* fresh) {
    uint32_t h = hslot<S>(key);
    *fresh = false;
    for (int probe = 0; probe < S; ++probe) {
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
    return (uint32_t)S;
}

template <typename OffT, typename ValT, bool NUMERIC>
__global__ void __launch_bounds__(RAP_WARPS * 32, 8) k_rap(int64_t mc, const OffT* __restrict__ rrm,
                                                      const int32_t* __restrict__ rent, const ValT* __restrict__ rval,
                                                      const OffT* __restrict__ arm, const int32_t* __restrict__ aent,
                                                      const ValT* __restrict__ aval, const OffT* __restrict__ prm,
                                                      const int32_t* __restrict__ pent, const ValT* __restrict__ pval,
                                                      int32_t* __restrict__ counts, const OffT* __restrict__ crm,
                                                      int32_t* __restrict__ cent, ValT* __restrict__ cval,
                                                      int* __restrict__ too_many) {
    __shared__ uint32_t skeys[RAP_WARPS][RAP_S];
    __shared__ ValT svals[NUMERIC ? RAP_WARPS : 1][NUMERIC ? RAP_S : 1];
    __shared__ uint32_t sstage[RAP_WARPS][RAP_CAP];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t* keys = skeys[warp];
    ValT* vals = svals[NUMERIC ? warp : 0];
    uint32_t* stage = sstage[warp];
    for (int t = lane; t < RAP_S; t += 32) {
        keys[t] = EMPTY;
        if (NUMERIC) vals[t] = (ValT)0;
    }
    __syncwarp();
    const int grp = lane >> 3, gl = lane & 7;  // 4 groups of 8 lanes
    const int64_t gw = (int64_t)blockIdx.x * RAP_WARPS + warp, nw = (int64_t)gridDim.x * RAP_WARPS;
    for (int64_t I = gw; I < mc; I += nw) {
        const int64_t rs = ld(rrm, I), re = ld(rrm, I + 1);
        int n = 0;  // distinct columns claimed (counted by the claiming lanes)
        bool full = false;
        // a lane's products come in runs of one column (the fine rows and neighbours of an
        // aggregate map to few coarse columns): a run is summed in registers and added to the
        // table once, which keeps most lanes off the same slot's compare-and-swap loop
        uint32_t run_c = EMPTY;
        ValT run_v = (ValT)0;
        auto flush = [&]() {
            if (run_c == EMPTY || full) return;
            bool fresh;
            const uint32_t h = rap_claim<RAP_S>(keys, run_c, &fresh);
            if (h == (uint32_t)RAP_S) {
                full = true;
                return;
            }
            n += fresh ? 1 : 0;
            if (NUMERIC) atomicAdd(&vals[h], run_v);
            run_c = EMPTY;
        };

        for (int64_t r0 = rs; r0 < re; r0 += 32) {
            const int nr = (int)min((int64_t)32, re - r0);
            int ii = 0;
            ValT rv = (ValT)0;
            if (lane < nr) {
                ii = __ldg(rent + r0 + lane);
                if (NUMERIC) rv = __ldg(rval + r0 + lane);
            }
            for (int t0 = 0; t0 < nr; t0 += 4) {
                const int t = t0 + grp;
                const int i = __shfl_sync(FULL, ii, min(t, nr - 1));
                const ValT r = __shfl_sync(FULL, rv, min(t, nr - 1));
                int64_t as = 0, ae = 0;
                if (t < nr) {
                    as = ld(arm, i);
                    ae = ld(arm, i + 1);
                }
                for (int64_t q = as + gl; q < ae; q += 8) {
                    const int j = __ldg(aent + q);
                    const ValT ra = NUMERIC ? r * __ldg(aval + q) : (ValT)0;
                    const int64_t ps = ld(prm, j), pe = ld(prm, j + 1);
                    for (int64_t u = ps; u < pe; ++u) {
                        const uint32_t c = (uint32_t)__ldg(pent + u);
                        const ValT v = NUMERIC ? ra * __ldg(pval + u) : (ValT)0;
                        if (c == run_c) {
                            run_v += v;  // same column as the lane's previous product
                        } else {
                            flush();
                            run_c = c;
                            run_v = v;
                        }
                    }
                }
            }
        }
        flush();
        __syncwarp();
        n = warp_sum(n);
        full = __any_sync(FULL, full);
        if (!NUMERIC) {
            if (lane == 0) counts[I] = n;
            if ((full || n > RAP_CAP) && lane == 0) atomicExch(too_many, 1);
            // reset the claimed slots
            for (int t = lane; t < RAP_S; t += 32) keys[t] = EMPTY;
            __syncwarp();
            continue;
        }
        // numeric epilogue: compaction, sort by column, coalesced write, reset
        const int64_t cb = ld(crm, I);
        const int clen = (int)(ld(crm, I + 1) - cb);
        int cnt = 0;
        uint32_t cmin = 0xffffffffu;
        for (int c0 = 0; c0 < RAP_S; c0 += 32) {
            const uint32_t kk = keys[c0 + lane];
            const bool occ = kk != EMPTY;
            const unsigned bal = __ballot_sync(FULL, occ);
            if (occ) {
                const int pos = cnt + __popc(bal & lanemask_lt());
                if (pos < RAP_CAP) stage[pos] = (uint32_t)(c0 + lane);
                cmin = min(cmin, kk);
            }
            cnt += __popc(bal);
        }
        cmin = __reduce_min_sync(FULL, cmin);
        __syncwarp();
        const int nn = min(min(cnt, clen), RAP_CAP);
        // keys (col - cmin) << 9 | slot, sorted by a warp bitonic sort sized to the row (E keys
        // per lane, 32E >= nn); columns spread over >= 2^23 sort the columns themselves
        auto sort_write = [&](auto EC) {
            constexpr int E = decltype(EC)::value;
            uint32_t v[E];
            bool wide = false;
#pragma unroll
            for (int q = 0; q < E; ++q) {
                const int idx = lane * E + q;
                if (idx < nn) {
                    const uint32_t sl = stage[idx];
                    const uint32_t d = keys[sl] - cmin;
                    wide |= d >= (1u << 23);
                    v[q] = (d << 9) | sl;
                } else {
                    v[q] = 0xffffffffu;
                }
            }
            const bool anywide = __any_sync(FULL, wide);
            if (anywide) {
#pragma unroll
                for (int q = 0; q < E; ++q) {
                    const int idx = lane * E + q;
                    v[q] = idx < nn ? keys[stage[idx]] : 0xffffffffu;
                }
            }
            warp_bitonic_sort<E>(v);
#pragma unroll
            for (int q = 0; q < E; ++q) {
                const int idx = lane * E + q;
                if (idx < nn) {
                    const uint32_t sl = anywide ? probe_find<RAP_S>(keys, v[q]) : (v[q] & (RAP_S - 1));
                    cent[cb + idx] = (int32_t)keys[sl];
                    cval[cb + idx] = vals[sl];
                }
            }
        };
        if (nn <= 32)
            sort_write(std::integral_constant<int, 1>{});
        else if (nn <= 64)
            sort_write(std::integral_constant<int, 2>{});
        else if (nn <= 128)
            sort_write(std::integral_constant<int, 4>{});
        else
            sort_write(std::integral_constant<int, 8>{});
        __syncwarp();
        for (int t = lane; t < RAP_S; t += 32) {
            keys[t] = EMPTY;
            vals[t] = (ValT)0;
        }
        __syncwarp();
    }
}

template <typename OffT, typename ValT, bool NUMERIC>
static void rap_t(Launch& L, const MatView& R, const MatView& A, const MatView& P, int32_t* counts, const void* crm,
                  int32_t* cent, void* cval, int* too_many) {
    if (R.nrows == 0) return;
    auto kern = k_rap<OffT, ValT, NUMERIC>;
    KCfg c = kernel_cfg(kern, RAP_WARPS * 32, 0, L.num_sms);
    const int grid = (int)std::min<int64_t>((R.nrows + RAP_WARPS - 1) / RAP_WARPS, c.grid_cap);
    L.begin(NUMERIC ? "rap_numeric" : "rap_symbolic", L.stream);
    kern<<<grid, RAP_WARPS * 32, 0, L.stream>>>(R.nrows, (const OffT*)R.row_map, R.entries, (const ValT*)R.values,
                                                (const OffT*)A.row_map, A.entries, (const ValT*)A.values,
                                                (const OffT*)P.row_map, P.entries, (const ValT*)P.values, counts,
                                                (const OffT*)crm, cent, (ValT*)cval, too_many);
    L.end(L.stream);
}

void rap_symbolic(Launch& L, bool off64, const MatView& R, const MatView& A, const MatView& P, int32_t* counts,
                  int* too_many) {
    if (off64)
        rap_t<int64_t, double, false>(L, R, A, P, counts, nullptr, nullptr, nullptr, too_many);
    else
        rap_t<int32_t, double, false>(L, R, A, P, counts, nullptr, nullptr, nullptr, too_many);
}

void rap_numeric(Launch& L, bool off64, bool f64, const MatView& R, const MatView& A, const MatView& P,
                 const void* crm, int32_t* cent, void* cval) {
    if (off64) {
        if (f64) rap_t<int64_t, double, true>(L, R, A, P, nullptr, crm, cent, cval, nullptr);
        else rap_t<int64_t, float, true>(L, R, A, P, nullptr, crm, cent, cval, nullptr);
    } else {
        if (f64) rap_t<int32_t, double, true>(L, R, A, P, nullptr, crm, cent, cval, nullptr);
        else rap_t<int32_t, float, true>(L, R, A, P, nullptr, crm, cent, cval, nullptr);
    }
}

}  // namespace kk

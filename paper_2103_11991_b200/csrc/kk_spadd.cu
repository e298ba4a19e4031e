// kk_spadd.cu -- SpAdd C = alpha A + beta B (Sec. 2.3), two phases.
//
// Symbolic (Alg. 1 "UnsortedSymbolic"): per row, the entries of A(i,:)
// and B(i,:) become keys (col, matrix, index) that are sorted by column; the unique
// columns are counted and every entry gets its scatter position Apos / Bpos in the row of
// C.  The paper's team bitonic sort becomes a warp bitonic sort of 64-bit keys held E per
// lane (rows with nnz(A_i) + nnz(B_i) <= 32E, E <= 8).  Sorted rows (checked per row) take
// the paper's sorted-input path: A's keys followed by B's in reverse form
// a bitonic sequence that the bitonic merge alone sorts (log2(32E) steps instead of the
// full sort's log2(32E)(log2(32E)+1)/2).  A row map scan follows (kk_setup.cu).
// Numeric: scatter alpha*a to Apos and beta*b to Bpos.  A warp owns a row
// and accumulates it in shared memory (entries of A or B with equal columns -- unmerged
// input -- add one at a time), then writes columns and values coalesced.
#include "kk_device.cuh"

namespace kk {

constexpr int SPADD_MAXE = 8;                   // keys per lane
constexpr int SPADD_MAXROW = 32 * SPADD_MAXE;   // nnz(A_i) + nnz(B_i) of the warp tier
// longer rows: a CTA per row, keys sorted in shared memory (block bitonic sort)
constexpr int SPADD_CTA_THREADS = 1024;
constexpr int SPADD_LONG_MAX = 16384;           // nnz(A_i) + nnz(B_i) limit of the CTA tier

// warp bitonic sort of 32*E 64-bit keys, E per lane (element e = lane*E + r)
template <int E>
__device__ __forceinline__ void warp_bitonic_sort64(unsigned long long (&v)[E]) {
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
                    const unsigned long long o = __shfl_xor_sync(FULL, v[r], lj);
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
                        const unsigned long long x = v[r], y = v[pr];
                        const bool sw = up ? (x > y) : (x < y);
                        v[r] = sw ? y : x;
                        v[pr] = sw ? x : y;
                    }
                }
            }
        }
    }
}

// the final merge of the bitonic sort: a bitonic sequence of 32*E keys (ascending then
// descending) sorted ascending in log2(32E) steps -- the paper's sorted-input SpAdd merge
// (A's entries followed by B's entries in reverse)
template <int E>
__device__ __forceinline__ void warp_bitonic_merge64(unsigned long long (&v)[E]) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int j = 16 * E; j > 0; j >>= 1) {
        if (j >= E) {
            const int lj = j / E;
#pragma unroll
            for (int r = 0; r < E; ++r) {
                const int e = lane * E + r;
                const unsigned long long o = __shfl_xor_sync(FULL, v[r], lj);
                v[r] = ((e & j) == 0) ? min(v[r], o) : max(v[r], o);
            }
        } else {
#pragma unroll
            for (int r = 0; r < E; ++r) {
                const int pr = r ^ j;
                if (pr > r) {
                    const unsigned long long x = v[r], y = v[pr];
                    v[r] = min(x, y);
                    v[pr] = max(x, y);
                }
            }
        }
    }
}

// key = col << 9 | matrix << 8 | index in its row (index < 256)
template <typename OffT, int E>
__global__ void __launch_bounds__(256) k_spadd_symbolic(int64_t m, const OffT* __restrict__ arm,
                                                        const int32_t* __restrict__ aent, const OffT* __restrict__ brm,
                                                        const int32_t* __restrict__ bent, int32_t* __restrict__ counts,
                                                        int32_t* __restrict__ apos, int32_t* __restrict__ bpos,
                                                        uint8_t* __restrict__ dup, int* __restrict__ too_long) {
    const int lane = threadIdx.x & 31;
    const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t i = gw; i < m; i += nw) {
        const int64_t sa = ld(arm, i), sb = ld(brm, i);
        const int na = (int)(ld(arm, i + 1) - sa), nb = (int)(ld(brm, i + 1) - sb);
        const int n = na + nb;
        // rows are taken by the smallest E that holds them
        if (n > 32 * E || (E > 1 && n <= 16 * E)) {
            continue;  // longer than the warp tier: k_spadd_symbolic_long
        }
        // A's keys ascending from position 0, B's from the end backwards, padding between:
        // with sorted rows this is a bitonic sequence and the merge alone sorts it
        unsigned long long v[E];
        constexpr int NP = 32 * E;
        bool ok = true;  // the sequence is bitonic (ascending, then descending)
#pragma unroll
        for (int r = 0; r < E; ++r) {
            const int e = lane * E + r;
            unsigned long long key = ~0ull;
            if (e < na)
                key = ((unsigned long long)(uint32_t)__ldg(aent + sa + e) << 9) | (unsigned long long)e;
            else if (e >= NP - nb)
                key = ((unsigned long long)(uint32_t)__ldg(bent + sb + (NP - 1 - e)) << 9) | 256ull |
                      (unsigned long long)(NP - 1 - e);
            v[r] = key;
        }
#pragma unroll
        for (int r = 0; r < E; ++r) {
            const int e = lane * E + r;
            const unsigned long long nx = r + 1 < E ? v[r + 1 < E ? r + 1 : r] : __shfl_down_sync(FULL, v[0], 1);
            if (e + 1 < na) ok &= v[r] <= nx;           // A ascending
            if (e >= NP - nb && e + 1 < NP) ok &= v[r] >= nx;  // B (reversed) descending
        }
        if (__all_sync(FULL, ok))
            warp_bitonic_merge64<E>(v);
        else
            warp_bitonic_sort64<E>(v);
        // heads of equal-column runs; a repeated (column, matrix) marks unmerged input
        const unsigned long long last_prev = __shfl_up_sync(FULL, v[E - 1], 1);
        int h[E];
        int cnt = 0;
        bool dp = false;
#pragma unroll
        for (int r = 0; r < E; ++r) {
            const int e = lane * E + r;
            const unsigned long long pv = r > 0 ? v[r - 1] : last_prev;
            const bool valid = e < n;
            h[r] = valid && (e == 0 || (pv >> 9) != (v[r] >> 9));
            dp |= valid && e > 0 && (pv >> 8) == (v[r] >> 8);
            cnt += h[r];
        }
        int x = cnt;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const int y = __shfl_up_sync(FULL, x, d);
            if (lane >= d) x += y;
        }
        int pos = x - cnt - 1;  // position of the run holding the element before this lane's first
#pragma unroll
        for (int r = 0; r < E; ++r) {
            const int e = lane * E + r;
            pos += h[r];
            if (e < n) {
                const int idx = (int)(v[r] & 255ull);
                if (v[r] & 256ull)
                    bpos[sb + idx] = pos;
                else
                    apos[sa + idx] = pos;
            }
        }
        const int total = __shfl_sync(FULL, x, 31);
        const bool anydup = __any_sync(FULL, dp);
        if (lane == 0) {
            counts[i] = total;
            dup[i] = anydup ? 1 : 0;
        }
    }
}

template <typename OffT, typename ValT>
__global__ void __launch_bounds__(256) k_spadd_numeric(int64_t m, ValT alpha, const OffT* __restrict__ arm,
                                                       const int32_t* __restrict__ aent, const ValT* __restrict__ aval,
                                                       ValT beta, const OffT* __restrict__ brm,
                                                       const int32_t* __restrict__ bent, const ValT* __restrict__ bval,
                                                       const OffT* __restrict__ crm, int32_t* __restrict__ cent,
                                                       ValT* __restrict__ cval, const int32_t* __restrict__ apos,
                                                       const int32_t* __restrict__ bpos, const uint8_t* __restrict__ dup) {
    __shared__ ValT sv[8][SPADD_MAXROW];
    __shared__ int32_t sc[8][SPADD_MAXROW];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    ValT* vals = sv[warp];
    int32_t* cols = sc[warp];
    const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t i = gw; i < m; i += nw) {
        const int64_t sa = ld(arm, i), sb = ld(brm, i), cb = ld(crm, i);
        const int na = (int)(ld(arm, i + 1) - sa), nb = (int)(ld(brm, i + 1) - sb);
        const int cn = (int)(ld(crm, i + 1) - cb);
        if (cn > SPADD_MAXROW) continue;  // symbolic refused the row
        const bool plain = dup[i] == 0;
        for (int t = lane; t < cn; t += 32) vals[t] = (ValT)0;
        __syncwarp();
        // A then B; without duplicates the positions of one matrix's row are distinct
        for (int side = 0; side < 2; ++side) {
            const int nn = side ? nb : na;
            const int64_t s0 = side ? sb : sa;
            const int32_t* en = side ? bent : aent;
            const ValT* va = side ? bval : aval;
            const int32_t* ps = side ? bpos : apos;
            const ValT sc_ = side ? beta : alpha;
            for (int q0 = 0; q0 < nn; q0 += 32) {
                const int q = q0 + lane;
                int p = 0;
                ValT w = (ValT)0;
                if (q < nn) {
                    p = __ldg(ps + s0 + q);
                    w = sc_ * __ldg(va + s0 + q);
                    cols[p] = __ldg(en + s0 + q);
                }
                if (plain) {
                    if (q < nn) vals[p] += w;
                } else {
                    // unmerged row: lanes of one column add in turn
                    for (int l = 0; l < 32; ++l) {
                        if (lane == l && q < nn) vals[p] += w;
                        __syncwarp();
                    }
                }
                __syncwarp();
            }
        }
        for (int t = lane; t < cn; t += 32) {
            cent[cb + t] = cols[t];
            cval[cb + t] = vals[t];
        }
        __syncwarp();
    }
}

// Rows with SPADD_MAXROW < nnz(A_i) + nnz(B_i) <= SPADD_LONG_MAX: a CTA owns the row (Alg. 1,
// PAPER.md:269-300, with the team sort as a block bitonic sort of 64-bit keys
// col << 32 | matrix << 31 | index in shared memory); heads of equal-column runs, their
// block-wide scan, Apos / Bpos and the count as in the warp tier.  Longer rows set too_long.
template <typename OffT>
__global__ void __launch_bounds__(SPADD_CTA_THREADS) k_spadd_symbolic_long(
    int64_t m, const OffT* __restrict__ arm, const int32_t* __restrict__ aent, const OffT* __restrict__ brm,
    const int32_t* __restrict__ bent, int32_t* __restrict__ counts, int32_t* __restrict__ apos,
    int32_t* __restrict__ bpos, uint8_t* __restrict__ dup, int* __restrict__ too_long) {
    extern __shared__ __align__(16) unsigned long long sk[];  // SPADD_LONG_MAX keys
    __shared__ int wsum[SPADD_CTA_THREADS / 32];
    __shared__ int sdup;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int64_t i = blockIdx.x; i < m; i += gridDim.x) {
        const int64_t sa = ld(arm, i), sb = ld(brm, i);
        const int64_t na = ld(arm, i + 1) - sa, nb = ld(brm, i + 1) - sb;
        const int64_t n = na + nb;
        if (n <= SPADD_MAXROW) continue;
        if (n > SPADD_LONG_MAX) {
            if (tid == 0) atomicExch(too_long, 1);
            continue;
        }
        int P = 1;
        while (P < n) P <<= 1;
        for (int e = tid; e < P; e += SPADD_CTA_THREADS) {
            unsigned long long key = ~0ull;
            if (e < na)
                key = ((unsigned long long)(uint32_t)__ldg(aent + sa + e) << 32) | (unsigned long long)e;
            else if (e < n)
                key = ((unsigned long long)(uint32_t)__ldg(bent + sb + (e - na)) << 32) | (1ull << 31) |
                      (unsigned long long)(e - na);
            sk[e] = key;
        }
        if (tid == 0) sdup = 0;
        __syncthreads();
        for (int k = 2; k <= P; k <<= 1) {
            for (int j = k >> 1; j > 0; j >>= 1) {
                for (int e = tid; e < P; e += SPADD_CTA_THREADS) {
                    const int pr = e ^ j;
                    if (pr > e) {
                        const unsigned long long x = sk[e], y = sk[pr];
                        const bool up = (e & k) == 0;
                        if (up ? (x > y) : (x < y)) {
                            sk[e] = y;
                            sk[pr] = x;
                        }
                    }
                }
                __syncthreads();
            }
        }
        // heads, their exclusive block scan (elements in contiguous chunks per thread)
        const int per = (P + SPADD_CTA_THREADS - 1) / SPADD_CTA_THREADS;
        const int e0 = tid * per, e1 = min(e0 + per, (int)n);
        int cnt = 0;
        bool dp = false;
        for (int e = e0; e < e1; ++e) {
            const unsigned long long v = sk[e];
            const bool h = e == 0 || (sk[e - 1] >> 32) != (v >> 32);
            dp |= e > 0 && (sk[e - 1] >> 31) == (v >> 31);
            cnt += h;
        }
        int x = cnt;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const int y = __shfl_up_sync(FULL, x, d);
            if (lane >= d) x += y;
        }
        if (lane == 31) wsum[warp] = x;
        if (dp) sdup = 1;
        __syncthreads();
        int base = 0, total = 0;
        for (int w = 0; w < SPADD_CTA_THREADS / 32; ++w) {
            if (w < warp) base += wsum[w];
            total += wsum[w];
        }
        int pos = base + x - cnt - 1;
        for (int e = e0; e < e1; ++e) {
            const unsigned long long v = sk[e];
            pos += (e == 0 || (sk[e - 1] >> 32) != (v >> 32)) ? 1 : 0;
            const int idx = (int)(v & 0x7fffffffull);
            if (v & (1ull << 31))
                bpos[sb + idx] = pos;
            else
                apos[sa + idx] = pos;
        }
        if (tid == 0) {
            counts[i] = total;
            dup[i] = sdup ? 1 : 0;
        }
        __syncthreads();
    }
}

// Numeric for the CTA-tier rows: scatter straight into C's row in global memory (columns
// stored, values zeroed, then alpha*a and beta*b added; fp64/fp32 reductions when the row
// has unmerged input, plain adds otherwise -- A's positions, then B's, are distinct)
template <typename OffT, typename ValT>
__global__ void __launch_bounds__(256) k_spadd_numeric_long(
    int64_t m, ValT alpha, const OffT* __restrict__ arm, const int32_t* __restrict__ aent,
    const ValT* __restrict__ aval, ValT beta, const OffT* __restrict__ brm, const int32_t* __restrict__ bent,
    const ValT* __restrict__ bval, const OffT* __restrict__ crm, int32_t* __restrict__ cent, ValT* __restrict__ cval,
    const int32_t* __restrict__ apos, const int32_t* __restrict__ bpos, const uint8_t* __restrict__ dup) {
    for (int64_t i = blockIdx.x; i < m; i += gridDim.x) {
        const int64_t cb = ld(crm, i), cn = ld(crm, i + 1) - cb;
        if (cn <= SPADD_MAXROW) continue;  // the warp tier's row
        const int64_t sa = ld(arm, i), sb = ld(brm, i);
        const int64_t na = ld(arm, i + 1) - sa, nb = ld(brm, i + 1) - sb;
        if (na + nb > SPADD_LONG_MAX) continue;
        const bool plain = dup[i] == 0;
        for (int64_t t = threadIdx.x; t < cn; t += blockDim.x) cval[cb + t] = (ValT)0;
        __syncthreads();
        for (int side = 0; side < 2; ++side) {
            const int64_t nn = side ? nb : na, s0 = side ? sb : sa;
            const int32_t* en = side ? bent : aent;
            const ValT* va = side ? bval : aval;
            const int32_t* ps = side ? bpos : apos;
            const ValT sc_ = side ? beta : alpha;
            for (int64_t q = threadIdx.x; q < nn; q += blockDim.x) {
                const int p = __ldg(ps + s0 + q);
                cent[cb + p] = __ldg(en + s0 + q);
                const ValT w = sc_ * __ldg(va + s0 + q);
                if (plain)
                    cval[cb + p] += w;
                else
                    atomicAdd(&cval[cb + p], w);
            }
            __syncthreads();
        }
    }
}

template <typename OffT>
static void spadd_symbolic_t(Launch& L, int64_t m, const MatView& A, const MatView& B, int32_t* counts,
                             int32_t* apos, int32_t* bpos, uint8_t* dup, int* too_long) {
    const int threads = 256;
    const int grid = (int)std::min<int64_t>((m * 32 + threads - 1) / threads, (int64_t)L.num_sms * 16);
    L.begin("spadd_symbolic", L.stream);
    k_spadd_symbolic<OffT, 1><<<grid, threads, 0, L.stream>>>(m, (const OffT*)A.row_map, A.entries, (const OffT*)B.row_map,
                                                              B.entries, counts, apos, bpos, dup, too_long);
    k_spadd_symbolic<OffT, 2><<<grid, threads, 0, L.stream>>>(m, (const OffT*)A.row_map, A.entries, (const OffT*)B.row_map,
                                                              B.entries, counts, apos, bpos, dup, too_long);
    k_spadd_symbolic<OffT, 4><<<grid, threads, 0, L.stream>>>(m, (const OffT*)A.row_map, A.entries, (const OffT*)B.row_map,
                                                              B.entries, counts, apos, bpos, dup, too_long);
    k_spadd_symbolic<OffT, 8><<<grid, threads, 0, L.stream>>>(m, (const OffT*)A.row_map, A.entries, (const OffT*)B.row_map,
                                                              B.entries, counts, apos, bpos, dup, too_long);
    {
        const size_t smem = (size_t)SPADD_LONG_MAX * 8;
        auto kern = k_spadd_symbolic_long<OffT>;
        KCfg c = kernel_cfg(kern, SPADD_CTA_THREADS, smem, L.num_sms);
        kern<<<std::min<int64_t>(m, c.grid_cap), SPADD_CTA_THREADS, smem, L.stream>>>(
            m, (const OffT*)A.row_map, A.entries, (const OffT*)B.row_map, B.entries, counts, apos, bpos, dup, too_long);
    }
    L.end(L.stream, 5);
}

void spadd_symbolic(Launch& L, bool off64, int64_t m, const MatView& A, const MatView& B, int32_t* counts,
                    int32_t* apos, int32_t* bpos, uint8_t* dup, int* too_long) {
    if (m == 0) return;
    if (off64)
        spadd_symbolic_t<int64_t>(L, m, A, B, counts, apos, bpos, dup, too_long);
    else
        spadd_symbolic_t<int32_t>(L, m, A, B, counts, apos, bpos, dup, too_long);
}

template <typename OffT, typename ValT>
static void spadd_numeric_t(Launch& L, int64_t m, double alpha, const MatView& A, double beta, const MatView& B,
                            const void* crm, int32_t* cent, void* cval, const int32_t* apos, const int32_t* bpos,
                            const uint8_t* dup) {
    const int threads = 256;
    const int grid = (int)std::min<int64_t>((m * 32 + threads - 1) / threads, (int64_t)L.num_sms * 8);
    L.begin("spadd_numeric", L.stream);
    k_spadd_numeric<OffT, ValT><<<grid, threads, 0, L.stream>>>(
        m, (ValT)alpha, (const OffT*)A.row_map, A.entries, (const ValT*)A.values, (ValT)beta, (const OffT*)B.row_map,
        B.entries, (const ValT*)B.values, (const OffT*)crm, cent, (ValT*)cval, apos, bpos, dup);
    k_spadd_numeric_long<OffT, ValT><<<(int)std::min<int64_t>(m, (int64_t)L.num_sms * 8), 256, 0, L.stream>>>(
        m, (ValT)alpha, (const OffT*)A.row_map, A.entries, (const ValT*)A.values, (ValT)beta, (const OffT*)B.row_map,
        B.entries, (const ValT*)B.values, (const OffT*)crm, cent, (ValT*)cval, apos, bpos, dup);
    L.end(L.stream, 2);
}

void spadd_numeric(Launch& L, bool off64, bool f64, int64_t m, double alpha, const MatView& A, double beta,
                   const MatView& B, const void* crm, int32_t* cent, void* cval, const int32_t* apos,
                   const int32_t* bpos, const uint8_t* dup) {
    if (m == 0) return;
    if (off64) {
        if (f64) spadd_numeric_t<int64_t, double>(L, m, alpha, A, beta, B, crm, cent, cval, apos, bpos, dup);
        else spadd_numeric_t<int64_t, float>(L, m, alpha, A, beta, B, crm, cent, cval, apos, bpos, dup);
    } else {
        if (f64) spadd_numeric_t<int32_t, double>(L, m, alpha, A, beta, B, crm, cent, cval, apos, bpos, dup);
        else spadd_numeric_t<int32_t, float>(L, m, alpha, A, beta, B, crm, cent, cval, apos, bpos, dup);
    }
}

}  // namespace kk

// kk_numeric.cuh -- numeric-phase pieces shared by the numeric translation units
// (kk_numeric.cu: hash / dense / hub / tiny tiers and the bin dispatch; kk_num_rank.cu:
// the pattern tiers).
#pragma once
#include "kk_device.cuh"

namespace kk {

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


// a7 for the rows whose pattern symbolic kept (numeric bins NUM_PAT_BIN0.. and
// NUM_PATH_BIN0..), kk_num_rank.cu
void launch_pattern_bins(Launch& L, const NumArgs& a);

// a7 for the dense bin (nnz(C_i) > 512) when k is wide enough for a column bit vector
// (kk_num_hub.cu); false: not applicable, the caller runs the windowed dense tier
bool launch_hub_bins(Launch& L, const NumArgs& a, cudaStream_t s);

}  // namespace kk

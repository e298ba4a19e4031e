// kk_num_rank.cu -- a7 + a8 for the rows whose compressed pattern the symbolic phase kept
// (Eq. 1, 174, 178): the output position of every product is its rank
// in the pattern, so the row is accumulated in a dense per-row value array and written
// sorted without a sort.
#include "kk_numeric.cuh"

#include <cstdlib>
#include <type_traits>

namespace kk {
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
// a7 for pattern rows, lean form (k_num_rank).  The method is k_num_pattern's -- the
// output position of a product is the rank of its column in the pattern kept by symbolic,
// rank(c) = prefix(word(c)) + popc(mask & bits below c), accum = + into a dense per-row
// value array (Eq. 1) -- with the per-product work cut down:
//   * dense word index (rows whose words span <= PAT_NWIN words): the prologue expands the
//     pattern into a slot table rtab[word index][bit] -> value slot, so a product's slot is
//     two dependent byte loads (word index, then rtab) and no popcount;
//   * value slots are the ranks scattered by slot(r) = (SLOT_MUL * r) mod M (M the smallest
//     prime above CAP), a bijection that breaks the arithmetic progressions of stencil
//     ranks: the 27 ranks of a 27-point B row are 9 runs of 3 at a fixed stride, which in
//     rank order put two lanes of a half-warp on one bank pair in every 8-byte access
//     (4.0 -> 3.2 wavefronts per access, offline bank simulation on C2 rows);
//   * each 32-entry A chunk becomes steps, one per 32-entry segment of its B rows (empty
//     B rows give none, a row of L entries ceil(L/32)), 16-byte records in windows of 32;
//   * steps are branch-free: lanes past the B row's end load a valid entry of it and
//     accumulate into a dump slot vals[NS], so no divergent region per step;
//   * two steps per iteration, loads two steps ahead, and both steps' slot lookups are
//     issued before either read-modify-write (the lookups only read the pattern tables);
//   * the epilogue writes entries and values coalesced, in rank order, from the slots.
// Needs B.nnz < 2^31 (32-bit element offsets) and strictly increasing B rows.
// HASHW: patterns whose words span more than PAT_NWIN words (wide rows, e.g. C5): the word
// index is a PAT_SW-slot hash of the words and (mask, prefix) per hash slot gives the rank
// by popcount (an rtab per hash slot would not fit); slots = ranks.
// ------------------------------------------------------------------------------------
template <int CAP>
struct RankPrime;
template <>
struct RankPrime<32> {
    static constexpr int M = 37;
};
template <>
struct RankPrime<64> {
    static constexpr int M = 67;
};
template <>
struct RankPrime<128> {
    static constexpr int M = 131;
};
template <>
struct RankPrime<256> {
    static constexpr int M = 257;
};
template <>
struct RankPrime<512> {
    static constexpr int M = 521;
};
constexpr uint32_t SLOT_MUL = 53;
#ifndef KK_RANK_DEP
#define KK_RANK_DEP 1
#endif

template <typename ValT, int CAP, bool HASHW = false>
struct RankLayout {
    static constexpr int NS = HASHW ? CAP : RankPrime<CAP>::M;  // value slots; slot NS: idle lanes
    using SlotT = typename std::conditional<(NS < 255), uint8_t, uint16_t>::type;
    static constexpr size_t vals = 0;                                                  // NS + 1 values
    static constexpr size_t cols = ((size_t)(NS + 1) * sizeof(ValT) + 15) / 16 * 16;  // column per slot
    static constexpr size_t rec = cols + ((size_t)NS * 4 + 15) / 16 * 16;             // 32 x {bb, len, a}
    // HASHW: (mask, prefix) per hash slot; dense: rtab[PAT_W][32] slots, then (word, mask)
    // per word index (the Jacobi insertion's pattern check)
    static constexpr size_t winfo = rec + 32 * 16;
    // rtab rows are RT = 36 entries apart (32 used): the 4-byte word holding (word index wi,
    // bit b) is 9*wi + b/4 (u8), so the rows of the ~9 words a B row touches spread over
    // the banks instead of landing on 4 bank groups (32-entry rows: bank = 8*wi + b/4)
    static constexpr uint32_t RT = 36;
    static constexpr size_t pw = winfo + (HASHW ? (size_t)PAT_SW * 8 : ((size_t)PAT_W * RT * sizeof(SlotT) + 15) / 16 * 16);
    static constexpr size_t widx = pw + (HASHW ? 0 : (size_t)PAT_W * 8);              // u8 index | hash keys
    static constexpr size_t bytes = (widx + (HASHW ? (size_t)PAT_SW * 4 : (size_t)PAT_NWIN) + 15) / 16 * 16;
    __device__ static __forceinline__ uint32_t slot(uint32_t r) {
        if constexpr (HASHW)
            return r;
        else
            return (SLOT_MUL * r) % (uint32_t)NS;
    }
};

template <typename OffT, typename ValT, int CAP, int MINB, bool HASHW, bool TEX = false>
__global__ void __launch_bounds__(256, MINB) k_num_rank(const OffT* __restrict__ arm, const int32_t* __restrict__ aent,
                                                        const ValT* __restrict__ aval, const OffT* __restrict__ brm,
                                                        const int32_t* __restrict__ bent, const ValT* __restrict__ bval,
                                                        const OffT* __restrict__ crm, int32_t* __restrict__ cent,
                                                        ValT* __restrict__ cval, const int32_t* __restrict__ perm,
                                                        const int* __restrict__ bin_start, int bin,
                                                        const uint2* __restrict__ pat, const long long* __restrict__ pat_off,
                                                        const int* __restrict__ pat_len, const ValT* __restrict__ dinv,
                                                        double omega, cudaTextureObject_t tb, cudaTextureObject_t tv) {
    using LY = RankLayout<ValT, CAP, HASHW>;
    using SlotT = typename LY::SlotT;
    constexpr uint32_t NS = (uint32_t)LY::NS;
    extern __shared__ __align__(16) unsigned char sm_rank[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, warps = blockDim.x >> 5;
    // all shared accesses as sm_rank + 32-bit offset (shared addressing, no generic)
    const uint32_t o_w = (uint32_t)warp * (uint32_t)LY::bytes;
    const uint32_t o_val = o_w + (uint32_t)LY::vals, o_col = o_w + (uint32_t)LY::cols;
    const uint32_t o_rec = o_w + (uint32_t)LY::rec, o_inf = o_w + (uint32_t)LY::winfo;
    const uint32_t o_pw = o_w + (uint32_t)LY::pw;
    const int r0 = bin_start[bin], r1 = bin_start[bin + 1];
    const int stride = gridDim.x * warps;
    int r = r0 + blockIdx.x * warps + warp;
    if (r >= r1) return;
    for (uint32_t t = lane; t <= NS; t += 32) *(ValT*)(sm_rank + o_val + t * (uint32_t)sizeof(ValT)) = (ValT)0;
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
        // ---- the row's pattern: word index, slot table (or (mask, prefix)), column per slot ----
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
        // word -> slot-table row: dense u8 index (row = word index), or the hash slot of the word
        uint32_t h0 = (uint32_t)lane, h1 = (uint32_t)lane + 32u;
        if constexpr (HASHW) {
            h0 = wt_insert(wkeys, p0.x, lane < pl);
            h1 = wt_insert(wkeys, p1.x, lane + 32 < pl);
        }
        auto expand = [&](uint2 p, uint32_t h, int pre) {
            if constexpr (HASHW) {
                *(uint2*)(sm_rank + o_inf + h * 8u) = make_uint2(p.y, (uint32_t)pre);
            } else {
                sm_rank[o_idx + p.x] = (uint8_t)h;
                if (dinv) *(uint2*)(sm_rank + o_pw + h * 8u) = p;
            }
            uint32_t m = p.y;
            uint32_t rk = (uint32_t)pre;
            while (m) {
                const uint32_t b = (uint32_t)(__ffs(m) - 1);
                const uint32_t sl = LY::slot(rk);
                *(int32_t*)(sm_rank + o_col + sl * 4u) = (int32_t)(p.x * 32u + b);
                if constexpr (!HASHW) *(SlotT*)(sm_rank + o_inf + (h * LY::RT + b) * (uint32_t)sizeof(SlotT)) = (SlotT)sl;
                m &= m - 1;
                ++rk;
            }
        };
        if (lane < pl) expand(p0, h0, pre0);
        if (lane + 32 < pl) expand(p1, h1, pre1);
        __syncwarp();
        // value slot of a column of the pattern
        auto slot_of = [&](int col, bool valid) -> uint32_t {
            uint32_t sl;
            if constexpr (HASHW) {
                const uint32_t w = (uint32_t)col >> 5;
                uint32_t wi = wt_slot(w);
                while (wkeys[wi] != w) wi = (wi + 1) & (PAT_SW - 1);  // present: no empty-slot test
                const uint2 mp = *(const uint2*)(sm_rank + o_inf + wi * 8u);
                sl = mp.y + __popc(mp.x & ~(0xffffffffu << (col & 31)));
            } else {
                const uint32_t wi = sm_rank[o_idx + ((uint32_t)col >> 5)];
                sl = *(const SlotT*)(sm_rank + o_inf + (wi * LY::RT + ((uint32_t)col & 31u)) * (uint32_t)sizeof(SlotT));
            }
            return valid ? sl : NS;
        };
        // idle lanes (past the B row's end) are predicated off: a common dump slot would sit
        // on the bank pair of real slots and cost a wavefront in the second half-warp
        auto acc = [&](uint32_t sl, ValT prod) {
            if (sl < NS) {
                ValT* q = (ValT*)(sm_rank + o_val + sl * (uint32_t)sizeof(ValT));
                *q += prod;
            }
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
                    if constexpr (TEX) {
                        // B through the texture pipe (its wavefronts are not the LSU's)
                        col = tex1Dfetch<int>(tb, q);
                        if constexpr (sizeof(ValT) == 8) {
                            const int2 v = tex1Dfetch<int2>(tv, q);
                            bv = (ValT)__hiloint2double(v.y, v.x);
                        } else {
                            bv = (ValT)tex1Dfetch<float>(tv, q);
                        }
                    } else {
                        col = __ldg(bent + q);
                        bv = __ldg(bval + q);
                    }
                    a = (ValT)__hiloint2double(rr.w, rr.z);
                };
                if constexpr (!HASHW) {
                    // one register set (the two-set form below spills here: 64 registers +
                    // 8 bytes of stack, num_rank 1.88 -> 2.10 ms on C2; at 3 CTAs per SM without
                    // the spill 2.15 ms)
                    int colA, colB;
                    ValT bA, bB, aA, aB;
                    bool vA, vB;
                    load(0, colA, bA, aA, vA);
                    load(1, colB, bB, aB, vB);
                    for (int t = 0; t < nt; t += 2) {
                        const uint32_t rA = slot_of(colA, vA), rB = slot_of(colB, vB);
                        const ValT pA = aA * bA, pB = aB * bB;
                        if (t + 2 < nt) {
                            // the next loads take the step index through an empty asm that
                            // consumes the products: the multiplies are issued first, so the
                            // fetches can target the registers they free
                            int t2 = t + 2;
                            if (KK_RANK_DEP) asm volatile("" : "+r"(t2) : "d"((double)pA), "d"((double)pB));
                            load(t2, colA, bA, aA, vA);
                            load(t2 + 1, colB, bB, aB, vB);
                        }
                        acc(rA, pA);
                        __syncwarp();
                        acc(rB, pB);
                        __syncwarp();
                    }
                    return;
                }
                // two register sets: the steps two ahead load into the set not being consumed,
                // so no loop-carried copy waits on the fetch it was just issued (with one set the
                // compiler moves the fetched value at the end of every iteration, which stalls
                // the iteration on the fetch: ncu, C2, 31 % of stall samples on that move;
                // C5 num_rank_hash 224.5 -> 210.5 ms)
                struct Step {
                    int col;
                    ValT b, a;
                    bool v;
                };
                Step x0, y0, x1, y1;
                load(0, x0.col, x0.b, x0.a, x0.v);
                load(1, y0.col, y0.b, y0.a, y0.v);
                auto half = [&](const Step& cA, const Step& cB, Step& nA, Step& nB, int tn) {
                    const uint32_t rA = slot_of(cA.col, cA.v), rB = slot_of(cB.col, cB.v);
                    const ValT pA = cA.a * cA.b, pB = cB.a * cB.b;
                    if (tn < nt) {
                        load(tn, nA.col, nA.b, nA.a, nA.v);
                        load(tn + 1, nB.col, nB.b, nB.a, nB.v);
                    }
                    acc(rA, pA);
                    __syncwarp();
                    acc(rB, pB);
                    __syncwarp();
                };
                for (int t = 0; t < nt; t += 4) {
                    half(x0, y0, x1, y1, t + 2);
                    if (t + 2 >= nt) break;
                    half(x1, y1, x0, y0, t + 4);
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
            // its slots (its columns lie in E's pattern when A(i,i) is stored).
            const ValT sc = (ValT)(-omega * (double)__ldg(dinv + i));
            for (int t = lane; t < clen; t += 32) {
                ValT* q = (ValT*)(sm_rank + o_val + LY::slot((uint32_t)t) * (uint32_t)sizeof(ValT));
                *q *= sc;
            }
            __syncwarp();
            const int bs = (int)ld(brm, i), bl = (int)(ld(brm, i + 1) - bs);
            for (int q0 = 0; q0 < bl; q0 += 32) {
                const bool valid = q0 + lane < bl;
                const int q = bs + min(q0 + lane, bl - 1);
                const int col = __ldg(bent + q);
                const uint32_t w = (uint32_t)col >> 5;
                // a column outside the pattern (A(i,i) not stored) must not land on a slot
                bool inpat;
                if constexpr (HASHW) {
                    // the word must be present before probing (no empty-slot test in slot_of)
                    uint32_t wi = wt_slot(w);
                    while (wkeys[wi] != w && wkeys[wi] != EMPTY) wi = (wi + 1) & (PAT_SW - 1);
                    inpat = wkeys[wi] == w && ((*(const uint2*)(sm_rank + o_inf + wi * 8u)).x >> (col & 31)) & 1u;
                } else {
                    // the dense index may hold a stale entry: check the indexed word itself
                    inpat = w - wb < (uint32_t)PAT_NWIN;
                    if (inpat) {
                        const uint32_t wi = sm_rank[o_idx + w];
                        const uint2 pwm = *(const uint2*)(sm_rank + o_pw + (wi & 63u) * 8u);
                        inpat = wi < (uint32_t)pl && pwm.x == w && ((pwm.y >> (col & 31)) & 1u);
                    }
                }
                acc(slot_of(inpat ? col : 0, valid && inpat), __ldg(bval + q));
                __syncwarp();
            }
        }
        // ---- entries and values in rank order, coalesced; reset ----
        if (HASHW) {
            if (lane < pl) wkeys[h0] = EMPTY;
            if (lane + 32 < pl) wkeys[h1] = EMPTY;
        }
        for (int t = lane; t < clen; t += 32) {
            const uint32_t sl = LY::slot((uint32_t)t);
            // C is written once and not read again here: streaming (evict-first) stores keep
            // L2 for B's rows, which neighbouring rows of C read again
            __stcs(cent + cb + t, *(const int32_t*)(sm_rank + o_col + sl * 4u));
            ValT* q = (ValT*)(sm_rank + o_val + sl * (uint32_t)sizeof(ValT));
            __stcs(cval + cb + t, *q);
            *q = (ValT)0;
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
    // B's entries and values through the texture pipe when the handle made texture objects
    // for them (C2: num_rank 1.97 -> 1.88 ms; the kernel is bound by the LSU's L1 data
    // wavefronts, and texture fetches are the TEX pipe's)
    const cudaTextureObject_t tb = a.tex_ent, tv = a.tex_val;
    const bool tex = tb != 0 && tv != 0;
    auto kern = tex ? k_num_rank<OffT, ValT, CAP, 4, HASHW, true> : k_num_rank<OffT, ValT, CAP, 4, HASHW, false>;
    KCfg c = kernel_cfg(kern, warps * 32, smem, L.num_sms);
    int64_t need = (rows + warps - 1) / warps;
    int grid = (int)std::min<int64_t>(need, c.grid_cap);
    L.begin(kname(HASHW ? "num_rank_hash" : "num_rank", CAP), L.stream);
    kern<<<grid, warps * 32, smem, L.stream>>>((const OffT*)a.A.row_map, a.A.entries, (const ValT*)a.A.values,
                                               (const OffT*)a.B.row_map, a.B.entries, (const ValT*)a.B.values,
                                               (const OffT*)a.c_row_map, a.c_entries, (ValT*)a.c_values, a.perm,
                                               a.bin_start, bin, a.pat, a.pat_off, a.pat_len, (const ValT*)a.dinv, a.omega,
                                               tb, tv);
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
    // 4 resident CTAs per SM (60 registers, no spills) measured fastest on C2
    auto kern = a.B.nnz >= INT32_MAX ? k_num_pattern<OffT, ValT, CAP, false, 4, DENSE>
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


template <typename OffT, typename ValT>
static void pattern_bins_t(Launch& L, const NumArgs& a) {
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

void launch_pattern_bins(Launch& L, const NumArgs& a) {
    if (a.off64) {
        if (a.f64) pattern_bins_t<int64_t, double>(L, a);
        else pattern_bins_t<int64_t, float>(L, a);
    } else {
        if (a.f64) pattern_bins_t<int32_t, double>(L, a);
        else pattern_bins_t<int32_t, float>(L, a);
    }
}

}  // namespace kk

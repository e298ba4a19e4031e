// kk_device.cuh -- device helpers and launch-config helpers shared by the kernel TUs.
//
// Product code only: nothing here is shared with oracle/ (DESIGN.md Sec. 2).
#pragma once
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
// launch configuration helpers
// ------------------------------------------------------------------------------------
struct KCfg {
    int threads;
    size_t smem;
    int grid_cap;  // max resident CTAs on the device
};


template <typename K>
inline KCfg kernel_cfg(K kern, int threads, size_t smem, int num_sms) {
    static std::mutex g_cfg_mu;
    static std::unordered_map<const void*, KCfg> g_cfg;
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
inline const char* kname(const char* base, int S) {
    static std::mutex mu;
    static std::unordered_map<std::string, std::string> names;
    std::lock_guard<std::mutex> lk(mu);
    std::string key = std::string(base) + "_S" + std::to_string(S);
    auto it = names.find(key);
    if (it == names.end()) it = names.emplace(key, key).first;
    return it->second.c_str();
}

// ------------------------------------------------------------------------------------
// warp-owned linear-probing tables with atomic-free claims (numeric strict, symbolic hash)
// ------------------------------------------------------------------------------------
// Probe position L in [0,S) (L = bank*R + row, R = S/32) -> slot row*32 + ((bank + 7*row) & 31).
// A key starts at bank = col & 31, row = hash(col >> 5): consecutive columns of one
// 32-column word sit in consecutive banks, and the 7*row rotation spreads keys of the
// same bank (e.g. stencil planes 32k columns apart) over different physical banks.
template <int S>
__device__ __forceinline__ uint32_t bm_slot(uint32_t L) {
    constexpr int R = S / 32, LOGR = ilog2(R);
    const uint32_t row = L & (R - 1);
    return row * 32u + (((L >> LOGR) + 7u * row) & 31u);
}

template <int S>
__device__ __forceinline__ uint32_t bm_start(uint32_t col) {
    constexpr int R = S / 32, LOGR = ilog2(R);
    return (col & 31u) * R + (((col >> 5) * 0x9E3779B1u) >> (32 - LOGR));
}

// Lane-local probe from position *L: stops at `col` or at an EMPTY slot; returns the key seen.
template <int S>
__device__ __forceinline__ uint32_t probe_local(const uint32_t* keys, uint32_t col, uint32_t& L, uint32_t& h) {
    uint32_t k = keys[h];
    while (k != col && k != EMPTY) {
        L = (L + 1) & (S - 1);
        h = bm_slot<S>(L);
        k = keys[h];
    }
    return k;
}

// Find or claim `col` for the lanes with act; returns the slot.  Keys of the active
// lanes may repeat (equal keys walk the same probe sequence and agree on the slot).
// Lanes probe on their own; lanes that reach an EMPTY slot write their key, the warp
// syncs, the lanes re-read, and a lane whose write lost probes on (rare).
template <int S>
__device__ __forceinline__ uint32_t strict_claim(uint32_t* keys, uint32_t col, bool act) {
    uint32_t L = bm_start<S>(col);
    uint32_t h = bm_slot<S>(L);
    bool need = false;
    if (act) need = probe_local<S>(keys, col, L, h) == EMPTY;
    if (need) keys[h] = col;
    __syncwarp();
    bool lost = false;
    if (need) lost = keys[h] != col;
    while (__any_sync(FULL, lost)) {
        __syncwarp();
        bool again = false;
        if (lost) {
            L = (L + 1) & (S - 1);
            h = bm_slot<S>(L);
            again = probe_local<S>(keys, col, L, h) == EMPTY;
            if (again) keys[h] = col;
        }
        __syncwarp();
        lost = again && keys[h] != col;
    }
    return h;
}

template <int S>
__device__ __forceinline__ uint32_t strict_find(const uint32_t* keys, uint32_t col) {
    uint32_t L = bm_start<S>(col);
    uint32_t h = bm_slot<S>(L);
    while (keys[h] != col) {
        L = (L + 1) & (S - 1);
        h = bm_slot<S>(L);
    }
    return h;
}

// ------------------------------------------------------------------------------------
// a5/a7 for tiny rows (flops_i <= TINY_MAX, so nnz(C_i) <= TINY_MAX): a lane owns a row
// and keeps its distinct columns (and values: accum = +) in a register list
// -- the paper's accumulator reduced to K registers.  Insert = unrolled compare against
// all K slots (empty slots hold INT_MAX, never a column); the row is sorted by an
// odd-even transposition network before it is written.
// ------------------------------------------------------------------------------------
template <int K, typename ValT, bool VALUES>
struct TinyList {
    int cols[K];
    ValT vals[K];
    int n;
    __device__ __forceinline__ TinyList() : n(0) {
#pragma unroll
        for (int k = 0; k < K; ++k) {
            cols[k] = INT_MAX;
            vals[k] = (ValT)0;
        }
    }
    __device__ __forceinline__ void insert(int c, ValT v) {
        bool found = false;
#pragma unroll
        for (int k = 0; k < K; ++k) {
            if (cols[k] == c) {
                if (VALUES) vals[k] += v;
                found = true;
            }
        }
        if (!found && n < K) {
#pragma unroll
            for (int k = 0; k < K; ++k) {
                if (k == n) {
                    cols[k] = c;
                    if (VALUES) vals[k] = v;
                }
            }
            ++n;
        }
    }
    __device__ __forceinline__ void scale(ValT s) {
#pragma unroll
        for (int k = 0; k < K; ++k) vals[k] *= s;
    }
    __device__ __forceinline__ void sort() {
#pragma unroll
        for (int rnd = 0; rnd < K; ++rnd) {
#pragma unroll
            for (int k = rnd & 1; k + 1 < K; k += 2) {
                const bool sw = cols[k] > cols[k + 1];
                const int c0 = cols[k], c1 = cols[k + 1];
                cols[k] = sw ? c1 : c0;
                cols[k + 1] = sw ? c0 : c1;
                if (VALUES) {
                    const ValT v0 = vals[k], v1 = vals[k + 1];
                    vals[k] = sw ? v1 : v0;
                    vals[k + 1] = sw ? v0 : v1;
                }
            }
        }
    }
};

}  // namespace kk

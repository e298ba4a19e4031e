// Microbenchmark: shared-memory wavefront grouping rules and SHFL cost on sm_100a.
// 4 CTAs/SM x 8 warps; each warp runs ITERS iterations of 8 independent accesses of one
// pattern; reports clocks per warp-access per SM (1.0 = one wavefront-equivalent per clock).
#include <cstdio>
#include <cuda_runtime.h>
#define ITERS 2048
#define U 8
template <int MODE>
__global__ void __launch_bounds__(256) kern(double* out, int salt) {
    __shared__ __align__(16) double sv[U * 256 + 64];
    for (int i = threadIdx.x; i < U * 256 + 64; i += blockDim.x) sv[i] = i;
    __syncthreads();
    const int lane = threadIdx.x & 31;
    unsigned idx = 0;
    if (MODE == 0) idx = lane;                                  // consecutive: ideal 2 wf
    if (MODE == 1) idx = (lane & 15) + 32 * (lane >> 4);         // halves on the same banks, other row
    if (MODE == 2) idx = (lane >> 1) + 32 * (lane & 1);          // lanes 2m,2m+1: same bank, other row
    if (MODE == 3) idx = (lane * 7) & 31;                        // permuted distinct
    if (MODE == 4) idx = (lane & 7) + 32 * (lane >> 3);          // 4 groups of 8 on 8 bank pairs
    if (MODE == 5) idx = lane;                                  // SHFL only
    if (MODE == 6) idx = lane;                                  // LDS.64 + SHFL
    if (MODE == 7) idx = 2 * lane;                              // LDS.128 consecutive (512 B)
    if (MODE == 8) idx = lane;                                  // LDS.32 consecutive
    if (MODE == 9) idx = (lane >> 1) + 64 * (lane & 1);          // LDS.32 pairs same bank
    if (MODE == 10) idx = lane;                                 // STS.64 consecutive
    if (MODE == 11) idx = (lane & 15) + 32 * (lane >> 4);        // STS.64 halves same banks
    if (MODE == 12) idx = (lane >> 1) + 32 * (lane & 1);         // STS.64 pairs same bank
    if (MODE == 13) idx = lane;                                 // LDS.U8 consecutive bytes
    double acc[U];
#pragma unroll
    for (int k = 0; k < U; ++k) acc[k] = 0;
    unsigned v[U];
#pragma unroll
    for (int k = 0; k < U; ++k) v[k] = lane + salt + k;
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int k = 0; k < U; ++k) {
            const unsigned o = idx + k * 256;
            if (MODE <= 4) acc[k] += sv[o];
            if (MODE == 5) v[k] = __shfl_sync(0xffffffffu, v[k], (lane + it + k) & 31);
            if (MODE == 6) { acc[k] += sv[o]; v[k] = __shfl_sync(0xffffffffu, v[k], (lane + it + k) & 31); }
            if (MODE == 7) { const double2 d = *(const double2*)&sv[o]; acc[k] += d.x * d.y; }
            if (MODE == 8 || MODE == 9) acc[k] += ((const float*)sv)[o];
            if (MODE >= 10 && MODE <= 12) sv[o] = acc[k] + it;
            if (MODE == 13) v[k] += ((const unsigned char*)sv)[o + (v[k] & 0x100)];
        }
        if (MODE >= 10) __syncwarp();
        idx ^= (unsigned)(acc[0] == -1.0);
    }
    double t = 0;
    unsigned tv = 0;
#pragma unroll
    for (int k = 0; k < U; ++k) { t += acc[k]; tv += v[k]; }
    if (t == -2.0 || tv == 0xdeadbeef) out[0] = t + tv + sv[lane];
}
int main() {
    cudaDeviceProp pr;
    cudaGetDeviceProperties(&pr, 0);
    int clk = 0;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    const int nsm = pr.multiProcessorCount;
    printf("%s SMs=%d clock=%d kHz\n", pr.name, nsm, clk);
    double* out;
    cudaMalloc(&out, 8);
    const char* names[] = {"LDS.64 consecutive", "LDS.64 halves share banks", "LDS.64 lane pairs share bank",
                           "LDS.64 permuted distinct", "LDS.64 4 groups of 8", "SHFL.32 only", "LDS.64 + SHFL",
                           "LDS.128 consecutive", "LDS.32 consecutive", "LDS.32 pairs same bank",
                           "STS.64 consecutive", "STS.64 halves share banks", "STS.64 pairs share bank", "LDS.U8 consecutive"};
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int mode = 0; mode < 14; ++mode) {
        float best = 1e9;
        for (int rep = 0; rep < 4; ++rep) {
            cudaEventRecord(a);
            switch (mode) {
#define L(M) case M: kern<M><<<nsm * 4, 256>>>(out, rep); break;
                L(0) L(1) L(2) L(3) L(4) L(5) L(6) L(7) L(8) L(9) L(10) L(11) L(12) L(13)
            }
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            if (ms < best) best = ms;
        }
        const double accesses = (double)nsm * 4 * 8 * ITERS * U;  // warp-accesses
        const double clk_per = (best * 1e-3) * (clk * 1e3) * nsm / accesses;
        printf("%-30s %8.3f ms  %.3f clk per warp-access per SM\n", names[mode], best, clk_per);
    }
    printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
}

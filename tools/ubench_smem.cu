// Microbenchmark: shared-memory RMW options for hash accumulators on sm_100a.
// Each kernel: 1 CTA per SM x 8 warps, every lane performs ITERS updates to
// pseudo-random distinct-per-warp-step slots of a shared array. Prints ns and
// updates/clk/SM for: plain f64 RMW, atomicAdd f64 (CAS loop), atomicAdd f32,
// atomicOr u32, atomicCAS u32, match_any + plain, global red.add.f64 (L2 resident).
#include <cstdio>
#include <cuda_runtime.h>
#define ITERS 4096
#define SLOTS 4096
__device__ __forceinline__ unsigned hsh(unsigned x){ x*=2654435761u; return x; }
template<int MODE>
__global__ void kern(double* out, double* gbuf, int gmask){
  __shared__ double sv[SLOTS];
  __shared__ unsigned sk[SLOTS];
  for(int i=threadIdx.x;i<SLOTS;i+=blockDim.x){sv[i]=0;sk[i]=0;}
  __syncthreads();
  int lane=threadIdx.x&31, warp=threadIdx.x>>5;
  unsigned base = warp*512;
  double acc=0;
  for(int it=0; it<ITERS; ++it){
    // distinct slots within a warp step: permutation of lanes
    unsigned s = base + ((lane*37u + it*97u) & 511u);
    double p = (double)(it&7) * 0.5;
    if(MODE==0){ sv[s] = sv[s] + p; __syncwarp(); }
    else if(MODE==1){ atomicAdd(&sv[s], p); }
    else if(MODE==2){ atomicAdd((float*)&sv[s], (float)p); }
    else if(MODE==3){ atomicOr(&sk[s], 1u<<(it&31)); }
    else if(MODE==4){ unsigned o = atomicCAS(&sk[s], 0u, (unsigned)it+1); acc += o; }
    else if(MODE==5){ unsigned m = __match_any_sync(0xffffffffu, s); if(__popc(m)==1) sv[s]=sv[s]+p; __syncwarp(); }
    else if(MODE==6){ atomicAdd(&gbuf[(blockIdx.x*8192 + (s*131u)) & gmask], p); }
    else if(MODE==7){ unsigned k = sk[s]; if(k==0xffffffffu) sk[s]=1; acc += k; }  // LDS + compare only
  }
  __syncthreads();
  double t=0; for(int i=threadIdx.x;i<SLOTS;i+=blockDim.x) t+=sv[i]+sk[i];
  if(t+acc==-1.0) out[0]=t;
}
int main(){
  int dev=0; cudaDeviceProp pr; cudaGetDeviceProperties(&pr,dev);
  int clk=0; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  printf("%s SMs=%d smemPerBlockOptin=%zu l2=%d clockkHz=%d\n", pr.name, pr.multiProcessorCount, pr.sharedMemPerBlockOptin, pr.l2CacheSize, clk);
  double* out; cudaMalloc(&out, 8); double* g; size_t gn = 1<<22; cudaMalloc(&g, gn*8); cudaMemset(g,0,gn*8);
  const char* names[]={"plain f64 RMW","atomicAdd f64 smem","atomicAdd f32 smem","atomicOr u32 smem","atomicCAS u32 smem","match_any+plain f64","red.add.f64 global(32MB)","LDS u32 only"};
  int nsm=pr.multiProcessorCount;
  cudaEvent_t a,b; cudaEventCreate(&a); cudaEventCreate(&b);
  for(int mode=0; mode<8; ++mode){
    for(int rep=0; rep<3; ++rep){
      cudaEventRecord(a);
      switch(mode){case 0:kern<0><<<nsm*2,256>>>(out,g,gn-1);break;case 1:kern<1><<<nsm*2,256>>>(out,g,gn-1);break;
        case 2:kern<2><<<nsm*2,256>>>(out,g,gn-1);break;case 3:kern<3><<<nsm*2,256>>>(out,g,gn-1);break;
        case 4:kern<4><<<nsm*2,256>>>(out,g,gn-1);break;case 5:kern<5><<<nsm*2,256>>>(out,g,gn-1);break;
        case 6:kern<6><<<nsm*2,256>>>(out,g,gn-1);break;case 7:kern<7><<<nsm*2,256>>>(out,g,gn-1);break;}
      cudaEventRecord(b); cudaEventSynchronize(b); float ms; cudaEventElapsedTime(&ms,a,b);
      double ups = (double)nsm*2*256*ITERS; double persmclk = ups/(ms*1e-3)/nsm/(1.9e9);
      if(rep==2) printf("%-28s %8.3f ms  %.2f updates/clk/SM (@1.9GHz)\n", names[mode], ms, persmclk);
    }
  }
  cudaError_t e=cudaGetLastError(); printf("err=%s\n", cudaGetErrorString(e));
}

// Round-2 microbenchmarks: FP64 op rates and integer/fp32-compare leaf variants.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s @%d\n",cudaGetErrorString(e),__LINE__); return 1;}}while(0)
struct __align__(16) Tab { double c[256]; float f[256]; };

__global__ void __launch_bounds__(256) dadd_peak(double* out, int iters, double a) {
  double x0=threadIdx.x, x1=x0+1, x2=x0+2, x3=x0+3, x4=x0+4, x5=x0+5, x6=x0+6, x7=x0+7;
  for (int i=0;i<iters;++i){
#pragma unroll
    for (int j=0;j<16;++j){ x0+=a; x1+=a; x2+=a; x3+=a; x4+=a; x5+=a; x6+=a; x7+=a;} }
  out[blockIdx.x*blockDim.x+threadIdx.x]=x0+x1+x2+x3+x4+x5+x6+x7;
}
// pure DSETP chain: compare against table constants, count via predicate popc-free add
__global__ void __launch_bounds__(256) dsetp2(const __grid_constant__ Tab t, double* out, int iters, int zmask) {
  double thr = 5.0 + (blockIdx.x*blockDim.x+threadIdx.x)*1e-7; unsigned cnt=0;
  for (int it=0; it<iters; ++it) {
    const double* tc = t.c + 2*(it & zmask);
#pragma unroll
    for (int s=0;s<256;++s) cnt += (tc[s] > thr) ? 0x01000000u : 0u;
    thr += 1e-6; }
  out[blockIdx.x*blockDim.x+threadIdx.x]=cnt;
}
template<int V>
__global__ void __launch_bounds__(256) leafV(const __grid_constant__ Tab t, double* out, int iters, int zmask) {
  double acc[9]; unsigned cnt[9];
  for (int i=0;i<9;++i){acc[i]=0;cnt[i]=0;}
  double thr = 5.0 + (blockIdx.x*blockDim.x+threadIdx.x)*1e-7;
  int zlo = threadIdx.x & zmask;
  for (int it=0; it<iters; ++it) {
    const double2* tc = reinterpret_cast<const double2*>(t.c) + (it & zmask);
    const float4* tf = reinterpret_cast<const float4*>(t.f) + (it & zmask);
    int thr_hi = __double2hiint(thr);
    float thr_f = (float)thr;
#pragma unroll
    for (int s4 = 0; s4 < 64; ++s4) {
      double2 ca = tc[2*s4], cb = tc[2*s4+1];
      float4 ff;
      if (V == 2) ff = tf[s4];
#pragma unroll
      for (int h = 0; h < 4; ++h) {
        const int s = 4*s4+h; const int cls = __popc(s);
        double c = h==0 ? ca.x : h==1 ? ca.y : h==2 ? cb.x : cb.y;
        unsigned mh;
        if (V == 0) {            // int hi-word compare, ISETP+SEL
          mh = (__double2hiint(c) > thr_hi) ? 0x01000000u : 0u;
        } else if (V == 1) {     // int subtract + PRMT sign replicate
          int d = thr_hi - __double2hiint(c);
          asm("prmt.b32 %0, %1, 0, 0x4B44;" : "=r"(mh) : "r"(d));
        } else {                 // fp32 compare
          float cf = h==0 ? ff.x : h==1 ? ff.y : h==2 ? ff.z : ff.w;
          mh = (cf > thr_f) ? 0x01000000u : 0u;
        }
        acc[cls] = fma(__hiloint2double((int)mh, zlo), c, acc[cls]);
        cnt[cls] += mh;
      }
    }
    thr += 1e-6; }
  double r=0; for (int i=0;i<9;++i) r += acc[i]*(cnt[i]>>16);
  out[blockIdx.x*blockDim.x+threadIdx.x] = r;
}

int main() {
  cudaDeviceProp prop; CK(cudaGetDeviceProperties(&prop, 0));
  int sms = prop.multiProcessorCount; int clk_khz=0; cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  double* out; CK(cudaMalloc(&out, sizeof(double)*sms*64*256));
  Tab t; for (int i=0;i<256;++i) { t.c[i] = 1.0 + (i*37 % 256)*0.04; t.f[i] = (float)t.c[i]; }
  cudaEvent_t e0,e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int grid = sms*8; float ms;
  dadd_peak<<<grid,256>>>(out, 10, 1e-9);
  cudaEventRecord(e0); dadd_peak<<<grid,256>>>(out, 4000, 1e-9); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
  cudaEventElapsedTime(&ms,e0,e1);
  printf("{\"kernel\":\"dadd_peak\",\"ms\":%.3f,\"dadd_per_s\":%.4e}\n", ms, (double)grid*256*4000*128/(ms*1e-3));
  dsetp2<<<grid,256>>>(t, out, 10, 0);
  cudaEventRecord(e0); dsetp2<<<grid,256>>>(t, out, 2000, 0); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
  cudaEventElapsedTime(&ms,e0,e1);
  printf("{\"kernel\":\"dsetp2\",\"ms\":%.3f,\"dsetp_per_s\":%.4e}\n", ms, (double)grid*256*2000*256/(ms*1e-3));
  for (int v=0; v<3; ++v) {
    auto launch=[&](int iters){ if(v==0) leafV<0><<<grid,256>>>(t,out,iters,0); else if(v==1) leafV<1><<<grid,256>>>(t,out,iters,0); else leafV<2><<<grid,256>>>(t,out,iters,0);};
    launch(10); cudaEventRecord(e0); launch(2000); cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); CK(cudaGetLastError());
    cudaEventElapsedTime(&ms,e0,e1);
    double lps = (double)grid*256*2000*256/(ms*1e-3);
    printf("{\"kernel\":\"leafV%d\",\"ms\":%.3f,\"leaves_per_s\":%.4e,\"warp_cycles_per_leaf_at_max\":%.3f}\n", v, ms, lps, (double)sms*4*32*(clk_khz*1e3)/lps);
  }
  return 0;
}

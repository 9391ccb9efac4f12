// Microbenchmarks for the exact-enumeration leaf loop design (tools/, not product).
// Measures FP64-pipe peak (DFMA), DSETP throughput, and two leaf-loop variants.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s @%d\n",cudaGetErrorString(e),__LINE__); return 1;}}while(0)

struct __align__(16) Tab { double c[256]; };

__global__ void __launch_bounds__(256) dfma_peak(double* out, int iters, double a, double b) {
  double x0=threadIdx.x, x1=x0+1, x2=x0+2, x3=x0+3, x4=x0+4, x5=x0+5, x6=x0+6, x7=x0+7;
  for (int i=0;i<iters;++i){
#pragma unroll
    for (int j=0;j<16;++j){ x0=fma(x0,a,b); x1=fma(x1,a,b); x2=fma(x2,a,b); x3=fma(x3,a,b);
      x4=fma(x4,a,b); x5=fma(x5,a,b); x6=fma(x6,a,b); x7=fma(x7,a,b);} }
  out[blockIdx.x*blockDim.x+threadIdx.x]=x0+x1+x2+x3+x4+x5+x6+x7;
}
__global__ void __launch_bounds__(256) dsetp_peak(double* out, int iters, double a, double b) {
  double x = threadIdx.x*1e-3; unsigned c0=0,c1=0,c2=0,c3=0;
  for (int i=0;i<iters;++i){
#pragma unroll
    for (int j=0;j<32;++j){ double t = a + j; c0 += (x > t); c1 += (x < t+0.5); c2 += (x>=t+0.25); c3 += (x<=t+0.75);} x += b; }
  out[blockIdx.x*blockDim.x+threadIdx.x]=c0+c1+c2+c3;
}
// variant A: constant-bank table, opaque uniform offset (LDCU.64 per leaf)
__global__ void __launch_bounds__(256) leafA(const __grid_constant__ Tab t, double* out, int iters, int zmask) {
  double acc[9]; unsigned cnt[9];
  for (int i=0;i<9;++i){acc[i]=0;cnt[i]=0;}
  double thr = 5.0 + (blockIdx.x*blockDim.x+threadIdx.x)*1e-7;
  int zlo = threadIdx.x & zmask;
  for (int it=0; it<iters; ++it) {
    const double2* tc = reinterpret_cast<const double2*>(t.c) + (it & zmask);
#pragma unroll
    for (int s2 = 0; s2 < 128; ++s2) {
      double2 cc = tc[s2];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int s = 2*s2+h; const int cls = __popc(s);
        double c = h ? cc.y : cc.x;
        unsigned mh = (c > thr) ? 0x01000000u : 0u;
        acc[cls] = fma(__hiloint2double((int)mh, zlo), c, acc[cls]);
        cnt[cls] += mh;
      }
    }
    thr += 1e-6; }
  double r=0; for (int i=0;i<9;++i) r += acc[i]*(cnt[i]>>24);
  out[blockIdx.x*blockDim.x+threadIdx.x] = r;
}
// variant B: shared-memory table (LDS.128 per 2 leaves)
__global__ void __launch_bounds__(256) leafB(const __grid_constant__ Tab t, double* out, int iters, int zmask) {
  __shared__ double2 sc[128];
  if (threadIdx.x < 128) sc[threadIdx.x] = make_double2(t.c[2*threadIdx.x], t.c[2*threadIdx.x+1]);
  __syncthreads();
  double acc[9]; unsigned cnt[9];
  for (int i=0;i<9;++i){acc[i]=0;cnt[i]=0;}
  double thr = 5.0 + (blockIdx.x*blockDim.x+threadIdx.x)*1e-7;
  int zlo = threadIdx.x & zmask;
  for (int it=0; it<iters; ++it) {
    const double2* tc = sc + (it & zmask);
#pragma unroll
    for (int s2 = 0; s2 < 128; ++s2) {
      double2 cc = tc[s2];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int s = 2*s2+h; const int cls = __popc(s);
        double c = h ? cc.y : cc.x;
        unsigned mh = (c > thr) ? 0x01000000u : 0u;
        acc[cls] = fma(__hiloint2double((int)mh, zlo), c, acc[cls]);
        cnt[cls] += mh;
      }
    }
    thr += 1e-6; }
  double r=0; for (int i=0;i<9;++i) r += acc[i]*(cnt[i]>>24);
  out[blockIdx.x*blockDim.x+threadIdx.x] = r;
}
// variant C: naive if-form (ptxas if-converts to DADD+FSEL)
__global__ void __launch_bounds__(256) leafC(const __grid_constant__ Tab t, double* out, int iters, int zmask) {
  double acc[9]; unsigned cnt[9];
  for (int i=0;i<9;++i){acc[i]=0;cnt[i]=0;}
  double thr = 5.0 + (blockIdx.x*blockDim.x+threadIdx.x)*1e-7;
  for (int it=0; it<iters; ++it) {
    const double* tc = t.c + 2*(it & zmask);
#pragma unroll
    for (int s = 0; s < 256; ++s) { const int cls = __popc(s); double c = tc[s];
      if (c > thr) { acc[cls] += c; cnt[cls] += 1; } }
    thr += 1e-6; }
  double r=0; for (int i=0;i<9;++i) r += acc[i]*cnt[i];
  out[blockIdx.x*blockDim.x+threadIdx.x] = r;
}

int main() {
  cudaDeviceProp prop; CK(cudaGetDeviceProperties(&prop, 0));
  int sms = prop.multiProcessorCount; int clk_khz=0; cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  printf("{\"gpu\":\"%s\",\"sms\":%d,\"clock_mhz\":%.0f}\n", prop.name, sms, clk_khz/1e3);
  double* out; CK(cudaMalloc(&out, sizeof(double)*sms*64*256));
  Tab t; for (int i=0;i<256;++i) t.c[i] = 1.0 + (i*37 % 256)*0.04;
  cudaEvent_t e0,e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int occ : {4, 8}) {
    int grid = sms*occ; float ms;
    int it = 4000;
    dfma_peak<<<grid,256>>>(out, 10, 1.0000001, 1e-9);
    cudaEventRecord(e0); dfma_peak<<<grid,256>>>(out, it, 1.0000001, 1e-9); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms,e0,e1);
    double ops = (double)grid*256*it*16*8;
    printf("{\"kernel\":\"dfma_peak\",\"occ\":%d,\"ms\":%.3f,\"dfma_per_s\":%.4e,\"per_sm_per_clk_at_max\":%.2f}\n", occ, ms, ops/(ms*1e-3), ops/(ms*1e-3)/sms/(clk_khz*1e3));
    dsetp_peak<<<grid,256>>>(out, 10, 1.0, 1e-9);
    cudaEventRecord(e0); dsetp_peak<<<grid,256>>>(out, it, 1.0, 1e-9); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms,e0,e1);
    ops = (double)grid*256*it*32*4;
    printf("{\"kernel\":\"dsetp\",\"occ\":%d,\"ms\":%.3f,\"cmp_per_s\":%.4e}\n", occ, ms, ops/(ms*1e-3));
    int li = 2000;
    for (int v=0; v<3; ++v) {
      auto launch=[&](int iters){ if(v==0) leafA<<<grid,256>>>(t,out,iters,0); else if(v==1) leafB<<<grid,256>>>(t,out,iters,0); else leafC<<<grid,256>>>(t,out,iters,0);};
      launch(10); cudaEventRecord(e0); launch(li); cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); CK(cudaGetLastError());
      cudaEventElapsedTime(&ms,e0,e1);
      double leaves = (double)grid*256*li*256;
      double lps = leaves/(ms*1e-3);
      printf("{\"kernel\":\"leaf%c\",\"occ\":%d,\"ms\":%.3f,\"leaves_per_s\":%.4e,\"warp_cycles_per_leaf_at_max\":%.3f}\n", 'A'+v, occ, ms, lps, (double)sms*4*32*(clk_khz*1e3)/lps);
    }
  }
  return 0;
}

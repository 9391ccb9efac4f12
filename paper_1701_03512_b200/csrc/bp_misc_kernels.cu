// K7: FP64-pipe peak microbenchmark (independent DFMA chains on every SM).
// MEASURED_PEAKS.json carries no FP64 figure, so bench.py measures it live.
#include "bp_kernels.h"

namespace bp {

__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// clk (optional): per CTA {SM cycles, ns} between the start and the end of
// its work, so the host can compute the SM clock the kernel actually ran at
__global__ void __launch_bounds__(256) k_dfma_peak(double* out, int iters, double a, double b,
                                                   unsigned long long* clk) {
  unsigned long long c0 = 0, t0 = 0;
  if (clk && threadIdx.x == 0) {
    c0 = clock64();
    t0 = global_ns();
  }
  double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6,
         x7 = x0 + 7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
      x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
  if (clk && threadIdx.x == 0) {
    clk[2 * blockIdx.x] = clock64() - c0;
    clk[2 * blockIdx.x + 1] = global_ns() - t0;
  }
}

cudaError_t launch_dfma_peak(double* out, int grid, int iters, cudaStream_t st, unsigned long long* clk) {
  k_dfma_peak<<<grid, 256, 0, st>>>(out, iters, 1.0000001, 1e-9, clk);
  return cudaGetLastError();
}

}  // namespace bp

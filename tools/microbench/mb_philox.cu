// Philox4x32-10 throughput on one B200 (design evidence for the MC kernel):
// blocks/s with S independent counter streams per thread, the same round
// function as the engine (csrc/bp_common.cuh).  Prints blocks/s, warp-cycles
// per block per SM sub-partition, and the Philox share of k_mc_strata's
// measured time.   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I ../../paper_1701_03512_b200/csrc
#include <cstdio>
#include "bp_common.cuh"

// the same generator with each 32x32 -> 64 product as two 32-bit halves
// (mul.hi.u32 + mul.lo.u32: IMAD.HI + IMAD instead of IMAD.WIDE)
__device__ __forceinline__ void philox_hilo(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3, uint32_t k0,
                                            uint32_t k1, uint32_t out[4]) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    uint32_t hi0, lo0, hi1, lo1;
    asm("mul.hi.u32 %0, %1, %2;" : "=r"(hi0) : "r"(c0), "r"(bp::kPhiloxM0));
    asm("mul.lo.u32 %0, %1, %2;" : "=r"(lo0) : "r"(c0), "r"(bp::kPhiloxM0));
    asm("mul.hi.u32 %0, %1, %2;" : "=r"(hi1) : "r"(c2), "r"(bp::kPhiloxM1));
    asm("mul.lo.u32 %0, %1, %2;" : "=r"(lo1) : "r"(c2), "r"(bp::kPhiloxM1));
    const uint32_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
    c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
    k0 += bp::kPhiloxW0;
    k1 += bp::kPhiloxW1;
  }
  out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

template <int S>
__global__ void __launch_bounds__(256) k_philox_hilo(unsigned iters, uint32_t key0, uint32_t key1, uint32_t* out) {
  uint32_t acc = 0;
  const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
  for (unsigned j = 0; j < iters; ++j) {
    uint32_t o[S][4];
#pragma unroll
    for (int s = 0; s < S; ++s) philox_hilo(j, tid, (uint32_t)s, 0u, key0, key1, o[s]);
#pragma unroll
    for (int s = 0; s < S; ++s) acc ^= o[s][0] ^ o[s][1] ^ o[s][2] ^ o[s][3];
  }
  out[tid] = acc;
}

template <int S>
void run_hilo(int sms, int clk_khz) {
  const int grid = sms * 8, threads = 256;
  const unsigned iters = 4096 / S;
  uint32_t* out;
  cudaMalloc(&out, sizeof(uint32_t) * grid * threads);
  k_philox_hilo<S><<<grid, threads>>>(16, 1, 2, out);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k_philox_hilo<S><<<grid, threads>>>(iters, 1, 2, out);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  const double per_s = (double)grid * threads * iters * S / (ms * 1e-3);
  printf("S=%d streams/thread, mul.hi + mul.lo halves: %.3e blocks/s, %.1f cycles per warp-block per SMSP\n", S,
         per_s, (double)sms * 4 * clk_khz * 1e3 / (per_s / 32));
  cudaFree(out);
}

template <int S, bool VKEY>
__global__ void __launch_bounds__(256) k_philox(unsigned iters, uint32_t key0, uint32_t key1, uint32_t* out) {
  uint32_t acc = 0;
  const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
  if (VKEY) {  // keys in vector registers (opaque per-thread zero) instead of uniform registers
    const uint32_t z = tid & (iters >> 30);
    key0 += z;
    key1 += z;
  }
  for (unsigned j = 0; j < iters; ++j) {
    uint32_t o[S][4];
#pragma unroll
    for (int s = 0; s < S; ++s) bp::philox4x32_10(j, tid, (uint32_t)s, 0u, key0, key1, o[s]);
#pragma unroll
    for (int s = 0; s < S; ++s) acc ^= o[s][0] ^ o[s][1] ^ o[s][2] ^ o[s][3];
  }
  out[tid] = acc;
}

template <int S, bool VKEY>
void run(int sms, int clk_khz) {
  const int grid = sms * 8, threads = 256;
  const unsigned iters = 4096 / S;
  uint32_t* out;
  cudaMalloc(&out, sizeof(uint32_t) * grid * threads);
  k_philox<S, VKEY><<<grid, threads>>>(16, 1, 2, out);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k_philox<S, VKEY><<<grid, threads>>>(iters, 1, 2, out);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  const double blocks = (double)grid * threads * iters * S;
  const double per_s = blocks / (ms * 1e-3);
  // warp-blocks per SMSP per cycle -> cycles per warp-block
  const double cyc = (double)sms * 4 * clk_khz * 1e3 / (per_s / 32);
  printf("S=%d streams/thread, keys in %s registers: %.3e blocks/s, %.1f cycles per warp-block per SMSP\n", S,
         VKEY ? "vector" : "uniform", per_s, cyc);
  cudaFree(out);
}

int main() {
  int sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  run<1, false>(sms, clk);
  run<2, false>(sms, clk);
  run<4, false>(sms, clk);
  run<1, true>(sms, clk);
  run<2, true>(sms, clk);
  run<4, true>(sms, clk);
  run_hilo<1>(sms, clk);
  run_hilo<2>(sms, clk);
  run_hilo<4>(sms, clk);
  // k_mc_strata (config 4): 2^28 draws x 13 blocks in 9.5 ms
  const double mc_blocks = 268435456.0 * 13 / 9.5e-3;
  printf("k_mc_strata runs %.3e Philox blocks/s (with the walk, payoff and Welford work around them)\n", mc_blocks);
  return 0;
}

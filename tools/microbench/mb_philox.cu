// Philox4x32-10 throughput on one B200 (design evidence for the MC kernel):
// blocks/s with S independent counter streams per thread, the same round
// function as the engine (csrc/bp_common.cuh).  Prints blocks/s, warp-cycles
// per block per SM sub-partition, and the Philox share of k_mc_strata's
// measured time.   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I ../../paper_1701_03512_b200/csrc
#include <cstdio>
#include "bp_common.cuh"

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
  // k_mc_strata (config 4): 2^28 draws x 13 blocks in 9.5 ms
  const double mc_blocks = 268435456.0 * 13 / 9.5e-3;
  printf("k_mc_strata runs %.3e Philox blocks/s (with the walk, payoff and Welford work around them)\n", mc_blocks);
  return 0;
}

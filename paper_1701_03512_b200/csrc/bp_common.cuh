// Shared device/host helpers for the binpaths B200 engine.
//
// * compensated (TwoSum / Neumaier-style) accumulation used by every
//   reduction, standing in for the reference's Kahan accumulator
//   (pkg/src/binpaths/exact.py:59-72);
// * fixed-order warp reductions (deterministic: the shuffle tree is the
//   same for every launch);
// * Philox4x32-10, the counter-based generator of the MC sampler
//   (replaces numpy Philox keyed by SeedSequence, mc.py:92-95).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#define BP_HD __host__ __device__ __forceinline__

namespace bp {

constexpr int kMaxN = 64;

// ---------------------------------------------------------------------------
// Compensated sums.  A pair (s, c) represents s + c.
// TwoSum (Knuth): exact error of one addition, branch free, 6 flops.
BP_HD void two_sum(double a, double b, double& s, double& e) {
  s = a + b;
  double bp = s - a;
  e = (a - (s - bp)) + (b - bp);
}
// add x into (s, c)
BP_HD void comp_add(double& s, double& c, double x) {
  double t, e;
  two_sum(s, x, t, e);
  s = t;
  c += e;
}
// merge (s2, c2) into (s, c)
BP_HD void comp_merge(double& s, double& c, double s2, double c2) {
  double t, e;
  two_sum(s, s2, t, e);
  s = t;
  c += c2 + e;
}

#ifdef __CUDACC__
// Fixed shuffle tree over a full warp; every lane ends with the total.
__device__ __forceinline__ void warp_comp_reduce(double& s, double& c) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    double s2 = __shfl_xor_sync(0xffffffffu, s, off);
    double c2 = __shfl_xor_sync(0xffffffffu, c, off);
    // order the operands by lane so lane pairs compute bit-identical sums
    const bool lo = ((threadIdx.x & 31) & off) == 0;
    double a_s = lo ? s : s2, a_c = lo ? c : c2;
    double b_s = lo ? s2 : s, b_c = lo ? c2 : c;
    comp_merge(a_s, a_c, b_s, b_c);
    s = a_s;
    c = a_c;
  }
}
#endif

// ---------------------------------------------------------------------------
// Philox4x32-10 (Salmon et al., SC'11), the same round function and
// constants as cuRAND's curand_Philox4x32_10.
constexpr uint32_t kPhiloxM0 = 0xD2511F53u;
constexpr uint32_t kPhiloxM1 = 0xCD9E8D57u;
constexpr uint32_t kPhiloxW0 = 0x9E3779B9u;
constexpr uint32_t kPhiloxW1 = 0xBB67AE85u;

BP_HD void philox_round(uint32_t& c0, uint32_t& c1, uint32_t& c2, uint32_t& c3,
                        uint32_t k0, uint32_t k1) {
  // one 32x32 -> 64 multiply per lane (IMAD.WIDE.U32 on the device)
  const uint64_t p0 = (uint64_t)kPhiloxM0 * c0;
  const uint64_t p1 = (uint64_t)kPhiloxM1 * c2;
  const uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
  const uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
  const uint32_t n0 = hi1 ^ c1 ^ k0;
  const uint32_t n2 = hi0 ^ c3 ^ k1;
  c0 = n0;
  c1 = lo1;
  c2 = n2;
  c3 = lo0;
}

BP_HD void philox4x32_10(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3,
                         uint32_t k0, uint32_t k1, uint32_t out[4]) {
#pragma unroll
  for (int r = 0; r < 9; ++r) {
    philox_round(c0, c1, c2, c3, k0, k1);
    k0 += kPhiloxW0;
    k1 += kPhiloxW1;
  }
  philox_round(c0, c1, c2, c3, k0, k1);
  out[0] = c0;
  out[1] = c1;
  out[2] = c2;
  out[3] = c3;
}

// The same block with the 10 round keys precomputed (rk[2 r], rk[2 r + 1];
// philox_round_keys on the host): the MC kernels read them straight from the
// parameter bank instead of running the key schedule once per block.
BP_HD void philox_round_keys(uint32_t k0, uint32_t k1, uint32_t rk[20]) {
  for (int r = 0; r < 10; ++r) {
    rk[2 * r] = k0;
    rk[2 * r + 1] = k1;
    k0 += kPhiloxW0;
    k1 += kPhiloxW1;
  }
}

BP_HD void philox4x32_10_rk(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3, const uint32_t (&rk)[20],
                            uint32_t out[4]) {
#pragma unroll
  for (int r = 0; r < 10; ++r) philox_round(c0, c1, c2, c3, rk[2 * r], rk[2 * r + 1]);
  out[0] = c0;
  out[1] = c1;
  out[2] = c2;
  out[3] = c3;
}

}  // namespace bp

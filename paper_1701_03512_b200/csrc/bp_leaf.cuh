// The explicit leaf block shared by the exact kernels (K1 bp_exact_kernels.cu,
// K3 bp_batch_kernels.cu).  See bp_exact.cuh for the math.
#pragma once
#include "bp_exact.cuh"

namespace bp {

// ---------------------------------------------------------------------------
// one explicit leaf test: n += (x OP th), as DSETP + predicated increment
template <bool GT>
__device__ __forceinline__ void leaf_test(int& n, double x, double th) {
  if (GT)
    asm("{.reg .pred p; setp.gt.f64 p, %1, %2; @p add.s32 %0, %0, 1;}" : "+r"(n) : "d"(x), "d"(th));
  else
    asm("{.reg .pred p; setp.lt.f64 p, %1, %2; @p add.s32 %0, %0, 1;}" : "+r"(n) : "d"(x), "d"(th));
}

// The leaf block of one table slot for NP nodes at once: every position i of
// the 2^L inner leaves is loaded once (uniform LDCU) and tested against each
// node's threshold; per group of <= kGroup the ITM count n selects the
// group's prefix sum.  acc[p][c] / cnt[p][c]: per-node, per-class ITM sum and
// count.  Compile-time recursion over (class C, group G): every index is constant.
template <int L, int NP, int SLOT, bool GT, int C, int G>
struct LeafGroups {
  static __device__ __forceinline__ void run(const double2* __restrict__ tb, const double* __restrict__ gpre,
                                             const double (&th)[NP], double (&acc)[NP][L + 1], int (&cnt)[NP][L + 1]) {
    if constexpr (C <= L) {
      constexpr int size = binom(L, C);
      if constexpr (kGroup * G < size) {
        constexpr int len = (size - kGroup * G) < kGroup ? (size - kGroup * G) : kGroup;
        constexpr int i0 = class_start(L, C) + kGroup * G;
        // the group's leaves count in independent chains of kChain (short
        // dependency chains); the in-the-money leaves of the group are a
        // prefix, so the sum of the chain counts indexes the group's prefix sums
        constexpr int NCH = (len + kChain - 1) / kChain;
        int nc[NP][NCH];
#pragma unroll
        for (int p = 0; p < NP; ++p)
#pragma unroll
          for (int c = 0; c < NCH; ++c) nc[p][c] = 0;
#pragma unroll
        for (int j = 0; j < len; ++j) {
          // 16-byte loads of positions (2k, 2k+1) of this slot's table
          const int i = SLOT * (1 << L) + i0 + j;
          const double2 v = tb[i >> 1];
          const double x = (i & 1) ? v.y : v.x;
#pragma unroll
          for (int p = 0; p < NP; ++p) leaf_test<GT>(nc[p][j / kChain], x, th[p]);
        }
        int n[NP];
#pragma unroll
        for (int p = 0; p < NP; ++p) {
          n[p] = 0;
#pragma unroll
          for (int c = 0; c < NCH; ++c) n[p] += nc[p][c];
        }
#pragma unroll
        for (int p = 0; p < NP; ++p) {
          acc[p][C] += gpre[(group_base(L, C) + G) * kGroupSlots + n[p]];
          cnt[p][C] += n[p];
        }
        LeafGroups<L, NP, SLOT, GT, C, G + 1>::run(tb, gpre, th, acc, cnt);
      } else {
        LeafGroups<L, NP, SLOT, GT, C + 1, 0>::run(tb, gpre, th, acc, cnt);
      }
    }
  }
};

template <int NP, int NC>
__device__ __forceinline__ void zero_acc(double (&acc)[NP][NC], int (&cnt)[NP][NC]) {
#pragma unroll
  for (int p = 0; p < NP; ++p)
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      acc[p][c] = 0.0;
      cnt[p][c] = 0;
    }
}

template <int L, int NP, int SLOT, bool GT>
__device__ __forceinline__ void leaf_block(const double2* __restrict__ tb, const double* __restrict__ gpre,
                                           const double (&th)[NP], double (&acc)[NP][L + 1], int (&cnt)[NP][L + 1]) {
  LeafGroups<L, NP, SLOT, GT, 0, 0>::run(tb, gpre, th, acc, cnt);
}

// K1: affine-threshold enumeration.  KM = compile-time kind mask.
}  // namespace bp

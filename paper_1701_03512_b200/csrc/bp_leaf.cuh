// The explicit leaf block shared by the exact kernels (K1 bp_exact_kernels.cu,
// K3 bp_batch_kernels.cu).  See bp_exact.cuh for the math.
#pragma once
#include "bp_exact.cuh"
#include "bp_gray.cuh"

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

// NP nodes' Gray counters over one group's operands: asm blocks of at most
// two nodes (bp_gray.cuh), all fed by the same table values
template <int LEN, bool GT, int NP>
__device__ __forceinline__ void gray_count(const double (&x)[LEN], const double (&th)[NP], unsigned (&off)[NP]) {
  if constexpr (NP <= 2) {
    GrayCount<LEN, GT, NP>::run(x, th, off);
  } else {
#pragma unroll
    for (int q = 0; q < NP; q += 2) {
      const double t2[2] = {th[q], th[q + 1]};
      unsigned o2[2];
      GrayCount<LEN, GT, 2>::run(x, t2, o2);
      off[q] = o2[0];
      off[q + 1] = o2[1];
    }
  }
}

// ---------------------------------------------------------------------------
// Gray-code leaf block.  Same explicit test per leaf (one FP64 compare), but
// the compare XORs its result into a predicate chain (bp_gray.cuh), so the
// count needs no instruction per leaf; per group and node the chains give a
// byte offset into the group's Gray-ordered table of {prefix sum, count}
// (kGraySlots 16-byte entries per group, gray_table_entry below).
constexpr int kGraySlots = gray_slots(kGroup);

// entry of Gray code g of a group from its prefix sums pre[0..kGroup]:
// {P[n], n} with n as the low word of .y (int counts) or as a double (fold)
__device__ inline double2 gray_table_entry(const double* pre, unsigned g, bool count_as_double) {
  unsigned n = g;
  for (int s = 1; s < 16; s <<= 1) n ^= n >> s;  // Gray -> binary
  if (n > (unsigned)kGroup) return make_double2(0.0, 0.0);
  return make_double2(pre[n], count_as_double ? (double)n : __longlong_as_double((long long)n));
}

template <int L, int NP, int SLOT, bool GT, int C, int G>
struct LeafGroupsGray {
  static __device__ __forceinline__ void run(const double2* __restrict__ tb, const char* __restrict__ gtab,
                                             const double (&th)[NP], double (&acc)[NP][L + 1], int (&cnt)[NP][L + 1]) {
    if constexpr (C <= L) {
      constexpr int size = binom(L, C);
      if constexpr (kGroup * G < size) {
        constexpr int len = (size - kGroup * G) < kGroup ? (size - kGroup * G) : kGroup;
        constexpr int i0 = class_start(L, C) + kGroup * G;
        double x[len];
#pragma unroll
        for (int j = 0; j < len; ++j) {
          const int i = SLOT * (1 << L) + i0 + j;
          const double2 v = tb[i >> 1];
          x[j] = (i & 1) ? v.y : v.x;
        }
        unsigned off[NP];
        gray_count<len, GT, NP>(x, th, off);
        const char* grp = gtab + (group_base(L, C) + G) * kGraySlots * kGrayEntry;
#pragma unroll
        for (int p = 0; p < NP; ++p) {
          const double2 e = *reinterpret_cast<const double2*>(grp + off[p]);
          acc[p][C] += e.x;
          cnt[p][C] += __double2loint(e.y);
        }
        LeafGroupsGray<L, NP, SLOT, GT, C, G + 1>::run(tb, gtab, th, acc, cnt);
      } else {
        LeafGroupsGray<L, NP, SLOT, GT, C + 1, 0>::run(tb, gtab, th, acc, cnt);
      }
    }
  }
};

template <int L, int NP, int SLOT, bool GT>
__device__ __forceinline__ void leaf_block_gray(const double2* __restrict__ tb, const char* __restrict__ gtab,
                                                const double (&th)[NP], double (&acc)[NP][L + 1],
                                                int (&cnt)[NP][L + 1]) {
  LeafGroupsGray<L, NP, SLOT, GT, 0, 0>::run(tb, gtab, th, acc, cnt);
}

// ---------------------------------------------------------------------------
// Gray leaf block with the class weights folded in as each class completes:
// per node only sA = sum_c w[h+c] A_c and sN = sum_c w[h+c] n_c stay live
// (A_c = sum of the class's in-the-money table values, n_c their count, both
// read from the Gray tables with n as a double).  The kinds' node values are
// affine in (sA, sN), see k_exact_fast.
template <int L, int NP, int SLOT, bool GT, int C, int G>
struct FoldGroups {
  static __device__ __forceinline__ void run(const double2* __restrict__ tb, const char* __restrict__ gtab,
                                             const double (&th)[NP], double (&A)[NP], double (&n)[NP]) {
    constexpr int size = binom(L, C);
    if constexpr (kGroup * G < size) {
      constexpr int len = (size - kGroup * G) < kGroup ? (size - kGroup * G) : kGroup;
      constexpr int i0 = class_start(L, C) + kGroup * G;
      double x[len];
#pragma unroll
      for (int j = 0; j < len; ++j) {
        const int i = SLOT * (1 << L) + i0 + j;
        const double2 v = tb[i >> 1];
        x[j] = (i & 1) ? v.y : v.x;
      }
      unsigned off[NP];
      gray_count<len, GT, NP>(x, th, off);
      const char* grp = gtab + (group_base(L, C) + G) * kGraySlots * kGrayEntry;
#pragma unroll
      for (int p = 0; p < NP; ++p) {
        const double2 e = *reinterpret_cast<const double2*>(grp + off[p]);
        A[p] = G == 0 ? e.x : A[p] + e.x;
        n[p] = G == 0 ? e.y : n[p] + e.y;
      }
      FoldGroups<L, NP, SLOT, GT, C, G + 1>::run(tb, gtab, th, A, n);
    }
  }
};

template <int L, int NP, int SLOT, bool GT, int C>
struct FoldClasses {
  static __device__ __forceinline__ void run(const double2* __restrict__ tb, const char* __restrict__ gtab,
                                             const double* __restrict__ sw, const int (&hn)[NP],
                                             const double (&th)[NP], double (&sA)[NP], double (&sN)[NP]) {
    if constexpr (C <= L) {
      double A[NP], n[NP];
      FoldGroups<L, NP, SLOT, GT, C, 0>::run(tb, gtab, th, A, n);
#pragma unroll
      for (int p = 0; p < NP; ++p) {
        const double w = sw[hn[p] + C];
        sA[p] = C == 0 ? w * A[p] : fma(w, A[p], sA[p]);
        sN[p] = C == 0 ? w * n[p] : fma(w, n[p], sN[p]);
      }
      FoldClasses<L, NP, SLOT, GT, C + 1>::run(tb, gtab, sw, hn, th, sA, sN);
    }
  }
};

template <int L, int NP, int SLOT, bool GT>
__device__ __forceinline__ void leaf_block_fold(const double2* __restrict__ tb, const char* __restrict__ gtab,
                                                const double* __restrict__ sw, const int (&hn)[NP],
                                                const double (&th)[NP], double (&sA)[NP], double (&sN)[NP]) {
  FoldClasses<L, NP, SLOT, GT, 0>::run(tb, gtab, sw, hn, th, sA, sN);
}

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

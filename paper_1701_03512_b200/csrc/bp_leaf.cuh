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
__host__ __device__ inline double2 gray_table_entry(const double* pre, unsigned g, bool count_as_double) {
  unsigned n = g;
  for (int s = 1; s < 16; s <<= 1) n ^= n >> s;  // Gray -> binary
  if (n > (unsigned)kGroup) return make_double2(0.0, 0.0);
  double y = (double)n;
  if (!count_as_double) {
    const long long v = (long long)n;
    std::memcpy(&y, &v, sizeof y);
  }
  return make_double2(pre[n], y);
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
// Gray-table group index of (class C, group 0): all classes, or (CMP) only the
// classes the I15 screen leaves to this block
template <int L, bool CMP>
__host__ __device__ constexpr int gray_group_base(int C) {
  if (!CMP) return group_base(L, C);
  int s = 0;
  for (int i = 0; i < C; ++i)
    if (!i15_class(L, i)) s += class_groups(L, i);
  return s;
}
template <int L>
__host__ __device__ constexpr int n_small_groups() { return gray_group_base<L, true>(L + 1); }

template <int L, int NP, int SLOT, bool GT, int C, int G, bool CMP = false>
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
      const char* grp = gtab + (gray_group_base<L, CMP>(C) + G) * kGraySlots * kGrayEntry;
#pragma unroll
      for (int p = 0; p < NP; ++p) {
        const double2 e = *reinterpret_cast<const double2*>(grp + off[p]);
        A[p] = G == 0 ? e.x : A[p] + e.x;
        n[p] = G == 0 ? e.y : n[p] + e.y;
      }
      FoldGroups<L, NP, SLOT, GT, C, G + 1, CMP>::run(tb, gtab, th, A, n);
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

// ---------------------------------------------------------------------------
// I15 screen of one big class for a node pair (node 0 in the low 16-bit lane,
// node 1 in the high lane).  Every leaf j is tested explicitly: one 32-bit
// multiply-add x_j * 1 + T forms, per lane, x~_j + 0x7FFF - theta~, whose
// bit 15 is set iff x~_j > theta~ (x~, theta~ = i15_map of the leaf value and
// of the node threshold, both <= 0x7FFF, so no carry crosses the lanes).  The
// result XORs into Gray-code counter bit ctz(j + 1) (the sorted class has its
// surely-in-the-money leaves as a prefix, so after the class the counters
// hold the Gray code of that prefix length n' per lane).  The code indexes
// the class's 32-byte entry {P_c[n'], n', x~_n' | P_c[m], x_n'}, m = the
// end of the tie run at n' (ExactArgs::te).  The only leaves whose
// screen is not decisive have x~ == theta~ and start at position n': a lane
// whose entry has x~_n' == theta~ tests leaf n' in fp64 (x_n' is in the
// entry; an in-the-money leaf takes its tie run with it) and, in the rarer
// case that position m has the same screened value too, walks on.
struct I15Ctx {
  const char* etab;          // the slot's entry table (shared memory)
  const unsigned* sxq;       // the slot's screened values (shared memory)
  const unsigned char* ste;  // the slot's tie-run ends (shared memory)
  unsigned one;         // 1, opaque to the compiler (keeps the multiply-add an IMAD)
  float thf[2];         // node thresholds in fp32
};
// bytes per entry: Asian slots {P[n'], n' | x~_n'}, {P[m], x_n'} (the rare fix
// reads m and x~_m from the tie-run and code arrays); lookback slots, whose
// fix runs for nearly every node, carry {P[n'], n' | x~_n'}, {P[m], m},
// {x_n', x~_m} so it needs no dependent loads
__host__ __device__ constexpr int i15_entry_bytes(bool lookback) { return lookback ? 48 : 32; }
#ifndef BP_I15_WAYS
#define BP_I15_WAYS 1  // r2 scan: 1 (no partials) best at 3 CTAs/SM, equal at 2
#endif
constexpr int kI15Ways = BP_I15_WAYS;  // partial Gray counters per bit

__host__ __device__ constexpr int ctz_c(int v) {
  int b = 0;
  while (!((v >> b) & 1)) ++b;
  return b;
}

// Where a slot's screen tables live: the kernel parameter block (K1: uniform
// constant-bank loads at compile-time offsets) or shared memory (K3: built by
// each CTA for its option).  i = class-major position, slot-relative.
template <int L, int SLOT>
struct ParamTabs {
  const ExactArgs<L>& a;
  const double* cp;  // the slot's class prefix sums (device image, global memory)
  __host__ __device__ __forceinline__ float nrm_s(int c) const { return a.nrm_s[SLOT][c]; }
  __host__ __device__ __forceinline__ float nrm_o(int c) const { return a.nrm_o[SLOT][c]; }
  __host__ __device__ __forceinline__ double tab(int i) const { return a.tab[SLOT * (1 << L) + i]; }
  __host__ __device__ __forceinline__ double cpre(int i) const { return cp[i]; }
};
struct SmemTabs {
  const float *ns, *no;
  const double *tb, *cp;
  const unsigned* xw;
  const unsigned char* tw;
  __host__ __device__ __forceinline__ float nrm_s(int c) const { return ns[c]; }
  __host__ __device__ __forceinline__ float nrm_o(int c) const { return no[c]; }
  __host__ __device__ __forceinline__ double tab(int i) const { return tb[i]; }
  __host__ __device__ __forceinline__ double cpre(int i) const { return cp[i]; }
  __host__ __device__ __forceinline__ unsigned xq(int i) const { return xw[i]; }
  __host__ __device__ __forceinline__ unsigned te(int i) const { return tw[i]; }
};

template <int L, int SLOT, bool GT, int C, class TS, bool FIXALL = false>
struct I15Class {
  static constexpr int len = binom(L, C), nb = bit_length(len), i0 = class_start(L, C);
  static __device__ __forceinline__ void run(const TS& a, const uint4* __restrict__ xb, const I15Ctx& x,
                                             const double (&th)[2], double (&A)[2], double (&n)[2]) {
    const float s = a.nrm_s(C), o = a.nrm_o(C);
    const unsigned k0 = i15_map(x.thf[0], s, o), k1 = i15_map(x.thf[1], s, o);
    const unsigned T = __byte_perm(0x7FFFu - k0, 0x7FFFu - k1, 0x5410);
    // counter bit b collects leaves j = 2^b - 1 + 2^(b+1) t; kI15Ways partial
    // counters per bit (by t) keep the XOR dependency chains short
    unsigned gp[nb][kI15Ways];
#pragma unroll
    for (int b = 0; b < nb; ++b)
#pragma unroll
      for (int q = 0; q < kI15Ways; ++q) gp[b][q] = 0u;
#pragma unroll
    for (int j = 0; j < len; ++j) {
      const uint4 w = xb[(i0 + j) >> 2];
      const int r = (i0 + j) & 3;
      const unsigned xv = r == 0 ? w.x : r == 1 ? w.y : r == 2 ? w.z : w.w;
      unsigned d;
      asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(xv), "r"(x.one), "r"(T));
      const int b = ctz_c(j + 1);
      gp[b][((j + 1) >> (b + 1)) % kI15Ways] ^= d;
    }
    unsigned g[nb];
#pragma unroll
    for (int b = 0; b < nb; ++b) {
      g[b] = gp[b][0];
#pragma unroll
      for (int q = 1; q < kI15Ways; ++q) g[b] ^= gp[b][q];
    }
    // byte offsets of the two lanes' codes: lane 1's bits (bit 31 of each
    // counter) shift in from the top, lane 0's (bit 15) are masked and added
    unsigned c1 = 0u, c0 = 0u;
#pragma unroll
    for (int b = nb - 1; b >= 0; --b) c1 = __funnelshift_l(g[b], c1, 1);
#pragma unroll
    for (int b = 0; b < nb; ++b) c0 += (g[b] & 0x8000u) << b;
    constexpr int EB = i15_entry_bytes(FIXALL);
    const char* et0 = x.etab + i15_base(L, C) * EB + (EB / 16) * (c0 >> 11);
    const char* et1 = x.etab + i15_base(L, C) * EB + (EB / 16) * (c1 << 4);
    const double2 e0 = *reinterpret_cast<const double2*>(et0);
    const double2 e1 = *reinterpret_cast<const double2*>(et1);
    double2 r0 = make_double2(e0.x, (double)__int_as_float(__double2loint(e0.y)));
    double2 r1 = make_double2(e1.x, (double)__int_as_float(__double2loint(e1.y)));
    const bool amb0 = (unsigned)__double2hiint(e0.y) == k0, amb1 = (unsigned)__double2hiint(e1.y) == k1;
    if constexpr (FIXALL) {
      // lookback kinds: nearly every node has a threshold tie in the class,
      // so every lane settles its boundary leaf without a branch
      fix_all(a, x, et0, th[0], k0, amb0, r0);
      fix_all(a, x, et1, th[1], k1, amb1, r1);
    } else if (__any_sync(__activemask(), amb0 || amb1)) {
      // warp-uniform branch (the surrounding control flow stays uniform; K3 may
      // run partial warps on tiny trees, hence the active mask)
      fix(a, x, et0, th[0], k0, amb0, r0);
      fix(a, x, et1, th[1], k1, amb1, r1);
    }
    A[0] = r0.x;
    n[0] = r0.y;
    A[1] = r1.x;
    n[1] = r1.y;
  }
  // fix without branches: loads and selects for every lane, the walk only
  // for a lane whose tie run ends on another leaf with the threshold's code
  static __device__ __forceinline__ void fix_all(const TS& a, const I15Ctx& x, const char* et, double th,
                                                 unsigned k, bool amb, double2& r) {
    const double2 q1 = *reinterpret_cast<const double2*>(et + 16);  // {P_c[m], m}
    const double2 q2 = *reinterpret_cast<const double2*>(et + 32);  // {x_n', x~_m}
    const bool itm = amb && (GT ? q2.x > th : q2.x < th);
    if (itm) r = q1;
    if (itm && (unsigned)__double2loint(q2.y) == k) r = walk(a, x, th, k, (int)q1.y);
  }
  // leaf n' in fp64 from the entry (with its tie run); a further leaf with
  // the threshold's screened value takes the exact walk
  static __device__ __forceinline__ void fix(const TS& a, const I15Ctx& x, const char* et, double th,
                                             unsigned k, bool amb, double2& r) {
    if (!amb) return;
    const double2 q1 = *reinterpret_cast<const double2*>(et + 16);  // {P_c[m], x_n'}
    if (GT ? q1.y > th : q1.y < th) {
      const int m = x.ste[i0 + (int)r.y];
      r = make_double2(q1.x, (double)m);
      if (m < len && (x.sxq[i0 + m] & 0xFFFFu) == k) r = walk(a, x, th, k, m);
    }
  }
  static __device__ __noinline__ double2 walk(const TS& a, const I15Ctx& x, double th, unsigned k, int j) {
    while (j < len && (x.sxq[i0 + j] & 0xFFFFu) == k) {
      const double v = a.tab(i0 + j);
      if (!(GT ? v > th : v < th)) break;
      j = x.ste[i0 + j];
    }
    return make_double2(a.cpre(i0 + C + j), (double)j);
  }
};

// K1 leaf block with the I15 screen on the big classes and the Gray fp64
// block (FoldGroups) on the others; per class the fold as leaf_block_fold.
template <int L, int SLOT, bool GT, int C, class TS, bool FIXALL = false>
struct FoldClassesI15 {
  static __device__ __forceinline__ void run(const TS& a, const uint4* __restrict__ xb, const I15Ctx& x,
                                             const double2* __restrict__ tb, const char* __restrict__ gtab,
                                             const double* __restrict__ sw, const int (&hn)[2],
                                             const double (&th)[2], double (&sA)[2], double (&sN)[2]) {
    if constexpr (C <= L) {
      double A[2], n[2];
      if constexpr (i15_class(L, C))
        I15Class<L, SLOT, GT, C, TS, FIXALL>::run(a, xb, x, th, A, n);
      else
        FoldGroups<L, 2, SLOT, GT, C, 0, true>::run(tb, gtab, th, A, n);
#pragma unroll
      for (int p = 0; p < 2; ++p) {
        const double w = sw[hn[p] + C];
        sA[p] = C == 0 ? w * A[p] : fma(w, A[p], sA[p]);
        sN[p] = C == 0 ? w * n[p] : fma(w, n[p], sN[p]);
      }
      FoldClassesI15<L, SLOT, GT, C + 1, TS, FIXALL>::run(a, xb, x, tb, gtab, sw, hn, th, sA, sN);
    }
  }
};

template <int L, int SLOT, bool GT, bool FIXALL = false, class TS>
__device__ __forceinline__ void leaf_block_fold_i15(const TS& a, const uint4* __restrict__ xb, I15Ctx x,
                                                    const double2* __restrict__ tb,
                                                    const char* __restrict__ gtab, const double* __restrict__ sw,
                                                    const int (&hn)[2], const double (&th)[2], double (&sA)[2],
                                                    double (&sN)[2]) {
  x.thf[0] = __double2float_rn(th[0]);
  x.thf[1] = __double2float_rn(th[1]);
  FoldClassesI15<L, SLOT, GT, 0, TS, FIXALL>::run(a, xb, x, tb, gtab, sw, hn, th, sA, sN);
}

// Quarter q of the entry for count n of class c (positions i0 .. i0+len),
// m = te(n), x~ of position len = 0xFFFF (never equal to a threshold):
//   Asian (32 B):    0 {P_c[n], n (fp32 bits) | x~_n << 32}, 1 {P_c[m], x_n}
//   lookback (48 B): 0 as above, 1 {P_c[m], m}, 2 {x_n, x~_m}
template <class TS>
__host__ __device__ inline double2 i15_quarter(const TS& a, int c, int i0, int len, int n, int q, bool lookback) {
  auto packed = [](unsigned hi, unsigned lo) {
    const unsigned long long b = ((unsigned long long)hi << 32) | lo;
    double d;
    memcpy(&d, &b, sizeof d);
    return d;
  };
  if (n > len) return make_double2(0.0, 0.0);
  const int m = n < len ? (int)a.te(i0 + n) : len;
  const unsigned xq_n = n < len ? (a.xq(i0 + n) & 0xFFFFu) : 0xFFFFu;
  const unsigned xq_m = m < len ? (a.xq(i0 + m) & 0xFFFFu) : 0xFFFFu;
  const double x_n = n < len ? a.tab(i0 + n) : 0.0;
  float nf = (float)n;
  unsigned nb;
  memcpy(&nb, &nf, sizeof nb);
  if (q == 0) return make_double2(a.cpre(i0 + c + n), packed(xq_n, nb));
  if (!lookback) return make_double2(a.cpre(i0 + c + m), x_n);
  if (q == 1) return make_double2(a.cpre(i0 + c + m), (double)m);
  return make_double2(x_n, packed(0u, xq_m));
}

// The slot's entry table, class by class (compile-time class layout): entry
// of Gray code g, n = gray^-1(g) <= |c|, is two 16-byte halves
// {P_c[n], n (fp32 bits) | x~_n << 32} and {P_c[te(n)], x_n}
// (x~_|c| = 0xFFFF: never equal to a threshold).
template <int L, int C, class TS>
__device__ inline void i15_fill(const TS& a, double2* __restrict__ et, bool lookback) {
  if constexpr (C <= L) {
    if constexpr (i15_class(L, C)) {
      constexpr int len = binom(L, C), i0 = class_start(L, C), base = i15_base(L, C), slots = i15_slots(L, C);
      const int nq = i15_entry_bytes(lookback) / 16;
      for (int t = threadIdx.x; t < nq * slots; t += blockDim.x) {
        unsigned n = (unsigned)(t / nq);
        for (int sh = 1; sh < 16; sh <<= 1) n ^= n >> sh;  // Gray -> binary
        et[nq * base + t] = i15_quarter(a, C, i0, len, (int)n, t % nq, lookback);
      }
    }
    i15_fill<L, C + 1, TS>(a, et, lookback);
  }
}

// the Gray tables of the classes the I15 screen leaves to the fp64 block
template <int L, int C>
__device__ inline void gray_fill_small(const double (*gpre)[kGroupSlots], double2* __restrict__ sg) {
  if constexpr (C <= L) {
    if constexpr (!i15_class(L, C)) {
      constexpr int ng = class_groups(L, C), dst = gray_group_base<L, true>(C), src = group_base(L, C);
      for (int i = threadIdx.x; i < ng * kGraySlots; i += blockDim.x)
        sg[dst * kGraySlots + i] = gray_table_entry(&gpre[src + i / kGraySlots][0], (unsigned)(i % kGraySlots), true);
    }
    gray_fill_small<L, C + 1>(gpre, sg);
  }
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

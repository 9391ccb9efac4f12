// K1 k_exact_fast: the affine-threshold class walk (see bp_exact.cuh).
// Kept in a header so build.py can compile one (L, kind-mask) instantiation
// per translation unit (bp_exact_fast_inst.cu) in parallel.
#pragma once
#include <cmath>
#include "bp_exact.cuh"
#include "bp_kernels.h"
#include "bp_leaf.cuh"



namespace bp {

// 1 / x without the library's out-of-range call (x is a positive normal node
// price): the MUFU estimate and two Newton steps (relative error ~1 ulp; the
// thresholds it feeds decide only leaves whose payoff is within rounding of 0)
__device__ __forceinline__ double fast_rcp(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0);
  r = fma(r, e, r);
  e = fma(-x, r, 1.0);
  return fma(r, e, r);
}


// resident CTAs per SM the register allocation targets: 3 for one table
// (<= 85 registers), 2 for the fused two-table kernels (measured best, r1)
__host__ __device__ constexpr int fast_tables(unsigned km) {
  return (int)((km >> kAC) & 1) + (int)((km >> kAP) & 1) + (int)((km >> kFL) & 1) + (int)((km >> kFLP) & 1);
}
#ifndef BP_MINB1
#define BP_MINB1 2  // resident CTAs per SM targeted by the one-table kernels (r2 scan at L = 9: 2 beats 3)
#endif
#ifndef BP_MINB2
#define BP_MINB2 2  // ... and by the fused two-table kernels
#endif
#ifndef BP_MINB_I15
#define BP_MINB_I15 2  // ... and by the one-table kernels of the Asian kinds (I15 screen; r2 scan: 2 beats 3 by 6 % at N=36)
#endif
// the table kind of slot 1 (kind order AC, AP, FL, FLP), 0 for one table
__host__ __device__ constexpr unsigned second_table_bit(unsigned km) {
  const int order[4] = {kAC, kAP, kFL, kFLP};
  bool seen = false;
  for (int i = 0; i < 4; ++i)
    if ((km >> order[i]) & 1) {
      if (seen) return 1u << order[i];
      seen = true;
    }
  return 0u;
}
#ifndef BP_SLOT_MAJOR
// two-table launches run slot-major: every warp's unit loop covers the units
// of slot 0's kinds, then those of slot 1's kind (one launch, one K2), so each
// stretch of the loop runs one slot's code and holds one slot's registers
#define BP_SLOT_MAJOR 1
#endif
#ifndef BP_K1_DYNAMIC
// units handed out by a counter (each warp's first unit is static): a warp
// that finishes early takes the next unit, so per-unit cost differences and
// per-SM speed differences do not set the kernel's tail
#define BP_K1_DYNAMIC 1
#endif

// One unit (2^(5 + m + L) paths) of K1 for the kinds KP of the launch's kind
// mask KM (the table slots and the shared-memory image are KM's); lane 0
// stores the unit's partial of every kind in KP.
template <int L, unsigned KM, unsigned KP, bool CNT>
__device__ __forceinline__ void fast_unit(const ExactArgs<L>& a, const double4* snib, const unsigned char* simg,
                                          const double* gcpre, unsigned long long unit, int lane,
                                          double2* __restrict__ unit_out, unsigned long long* shist,
                                          unsigned long long& leaves, unsigned long long& code_sum) {
  constexpr int NC = L + 1;
  constexpr bool kAC_ = (KP >> kAC) & 1, kAP_ = (KP >> kAP) & 1, kFL_ = (KP >> kFL) & 1,
                 kFLP_ = (KP >> kFLP) & 1, kEC_ = (KP >> kEC) & 1, kEP_ = (KP >> kEP) & 1;
  constexpr bool needMx = kFL_, needMn = kFLP_;
  // table slots of the launch (KM) in kind order AC, AP, FL, FLP
  constexpr bool mAC = (KM >> kAC) & 1, mAP = (KM >> kAP) & 1, mFL = (KM >> kFL) & 1;
  constexpr int slotAC = 0, slotAP = (int)mAC, slotFL = (int)mAC + (int)mAP, slotFLP = slotFL + (int)mFL;
  constexpr int NP = kNodesPerBlock;
  constexpr K1SmemLayout LY = k1_smem_layout<L>(KM);
  const double* sw = reinterpret_cast<const double*>(simg + LY.sw);
  const double* sW1 = reinterpret_cast<const double*>(simg + LY.sW1);
  const double* sW2 = reinterpret_cast<const double*>(simg + LY.sW2);
  const ExactScalars& sc = a.s;
  const double INF = __longlong_as_double(0x7ff0000000000000ll);
#define BP_GTAB(SLOT) reinterpret_cast<const char*>(simg + LY.sgray[SLOT])
  double ts[kNumKinds], tc[kNumKinds];
#pragma unroll
  for (int k = 0; k < kNumKinds; ++k) { ts[k] = 0.0; tc[k] = 0.0; }
 for (unsigned long long rr = 0; rr < (1ull << sc.q); ++rr) {
  const unsigned long long tp = (((unit << sc.q) | rr) << 5) | (unsigned long long)lane;  // thread prefix, Dp bits
  // --- prefix walk: steps 1..Dp (reference asset_path, model.py:164-172):
  // the first Dp mod 4 steps one by one, then four steps per nibble-table
  // lookup (relative price after the nibble, sum, max and min of its
  // relative prices)
  double S = sc.S0, Sig = 0.0, Mx = 0.0, Mn = INF;
  int h = 0;
  int t = sc.Dp - 1;
  for (; t >= 0 && ((t + 1) & 3); --t) {
    const int b = (int)((tp >> t) & 1ull);
    S *= b ? sc.u : sc.d;
    Sig += S;
    if (needMx) Mx = fmax(Mx, S);
    if (needMn) Mn = fmin(Mn, S);
    h += b;
  }
  for (; t >= 3; t -= 4) {
    const int nb = (int)((tp >> (t - 3)) & 15ull);
    const double4 q = snib[nb];  // {e, c, mx, mn}
    Sig = fma(S, q.y, Sig);
    if (needMx) Mx = fmax(Mx, S * q.z);
    if (needMn) Mn = fmin(Mn, S * q.w);
    S *= q.x;
    h += __popc(nb);
  }

  // nodes are processed NP at a time (n_mid is a multiple of NP: m >= 1)
  for (int j0 = 0; j0 < sc.n_mid; j0 += NP) {
    // table offset 0, opaque (the loads stay inside the loop) and, as a
    // warp reduction, held in a uniform register (uniform LDCU loads)
    const int zoff = (int)__reduce_or_sync(0xffffffffu, (unsigned)(j0 & sc.zero));
    double Sn[NP], Sg[NP], Mxn[NP], Mnn[NP], base[NP], thC[NP], thX[NP], thN[NP];
    int hn[NP];
#pragma unroll
    for (int p = 0; p < NP; ++p) {
      // --- node state at depth D
      const int j = j0 + p;
      Sn[p] = S * a.mid_e[j];
      Sg[p] = fma(S, a.mid_c[j], Sig);
      Mxn[p] = needMx ? fmax(Mx, S * a.mid_mx[j]) : 0.0;
      Mnn[p] = needMn ? fmin(Mn, S * a.mid_mn[j]) : 0.0;
      hn[p] = h + a.mid_h[j];
      base[p] = Sg[p] - sc.NK;
      const double rS = fast_rcp(Sn[p]);
      thC[p] = (kAC_ || kAP_) ? -base[p] * rS : 0.0;
      thX[p] = kFL_ ? Mxn[p] * rS : 0.0;
      thN[p] = kFLP_ ? fmin(Mnn[p], sc.K) * rS : 0.0;
    }

    const double2* tb = reinterpret_cast<const double2*>(a.tab) + zoff;  // + 0, opaque
    // --- per kind: the leaf block (2^L explicit leaf tests per node), then
    // the class finalisation, node value = sum_c w[h+c] * contrib_c.  Kinds
    // run one after the other so only one kind's accumulators are live.
    // the leaf block of a slot: the I15 screen where the layout puts it (the
    // lookback slots fix every lane's boundary leaf without a branch)
#define BP_FOLDLEAF(SLOT, GTV, TH)                                                                            \
if constexpr (LY.i15[SLOT])                                                                                \
  leaf_block_fold_i15<L, SLOT, GTV, LY.lookback[SLOT]>(                                                    \
      ParamTabs<L, SLOT>{a, gcpre + (SLOT) * ((1 << L) + L + 1)},                                          \
      reinterpret_cast<const uint4*>(simg + LY.sxq[SLOT]) + zoff,                                          \
      I15Ctx{reinterpret_cast<const char*>(simg + LY.si15[SLOT]),                                          \
             reinterpret_cast<const unsigned*>(simg + LY.sxq[SLOT]), simg + LY.ste[SLOT],                 \
             1u | (unsigned)sc.zero, {0.f, 0.f}},                                                          \
      tb, BP_GTAB(SLOT), sw, hn, TH, sA, sN);                                                              \
else                                                                                                       \
  leaf_block_fold<L, NP, SLOT, GTV>(tb, BP_GTAB(SLOT), sw, hn, TH, sA, sN)
    // node value, affine in sA = sum_c w[h+c] A_c and sN = sum_c w[h+c] n_c
    // (A_c / n_c: class-c in-the-money table sum and count):
    //   AC  S sA + base sN              AP  -(S sA + base sN)
    //   FL  S (sA - W2) + Mx (W1 - sN)  FLP K sN - S sA + max(K - Mn, 0) (W1 - sN)
    if constexpr (kAC_ || kAP_) {
      double sA[NP], sN[NP];
      if constexpr (kAC_) {
        BP_FOLDLEAF(slotAC, true, thC);
      } else {
        BP_FOLDLEAF(slotAP, false, thC);
      }
#pragma unroll
      for (int p = 0; p < NP; ++p) {
        const double v = fma(Sn[p], sA[p], base[p] * sN[p]);
        if (kAC_) comp_add(ts[kAC], tc[kAC], v);
        else comp_add(ts[kAP], tc[kAP], -v);
      }
    }
    if constexpr (kFL_) {
      double sA[NP], sN[NP];
      BP_FOLDLEAF(slotFL, true, thX);
#pragma unroll
      for (int p = 0; p < NP; ++p)
        comp_add(ts[kFL], tc[kFL], fma(Sn[p], sA[p] - sW2[hn[p]], Mxn[p] * (sW1[hn[p]] - sN[p])));
    }
    if constexpr (kFLP_) {
      double sA[NP], sN[NP];
      BP_FOLDLEAF(slotFLP, false, thN);
#pragma unroll
      for (int p = 0; p < NP; ++p) {
        const double flat = fmax(sc.K - Mnn[p], 0.0);
        comp_add(ts[kFLP], tc[kFLP], fma(flat, sW1[hn[p]] - sN[p], fma(sc.K, sN[p], -Sn[p] * sA[p])));
      }
    }
    if (kEC_ || kEP_) {
#pragma unroll
      for (int p = 0; p < NP; ++p) {
        double vEC = 0.0, vEP = 0.0;
#pragma unroll
        for (int c = 0; c < NC; ++c) {
          const double wv = sw[hn[p] + c], bc = a.b_cls[c];
          if (kEC_) vEC = fma(wv, bc * fmax(fma(Sn[p], a.e_cls[c], -sc.K), 0.0), vEC);
          if (kEP_) vEP = fma(wv, bc * fmax(fma(-Sn[p], a.e_cls[c], sc.K), 0.0), vEP);
        }
        if (kEC_) comp_add(ts[kEC], tc[kEC], vEC);
        if (kEP_) comp_add(ts[kEP], tc[kEP], vEP);
      }
    }

    if (CNT) {
#pragma unroll
      for (int p = 0; p < NP; ++p) {
        // leaf bookkeeping (K6): leaves per total up count, code coverage
        const unsigned long long node = (tp << sc.m) | (unsigned long long)(j0 + p);
#pragma unroll
        for (int c = 0; c < NC; ++c) atomicAdd(&shist[hn[p] + c], (unsigned long long)binom(L, c));
        leaves += 1ull << L;
        // sum of codes node*2^L + s, s < 2^L
        code_sum += (node << (2 * L)) + (((1ull << L) * ((1ull << L) - 1)) >> 1);
      }
    }
  }
 }  // rr
  // --- per-unit partial: fixed warp tree, lane 0 stores
#pragma unroll
  for (int k = 0; k < kNumKinds; ++k) {
    if (!((KP >> k) & 1)) continue;
    double s = ts[k], c = tc[k];
    warp_comp_reduce(s, c);
    if (lane == 0) unit_out[unit * kNumKinds + k] = make_double2(s, c);
  }
}
#undef BP_GTAB
#undef BP_FOLDLEAF

template <int L, unsigned KM, bool CNT>
__global__ void __launch_bounds__(256, fast_tables(KM) == 2                                      ? BP_MINB2
                                       : (i15_on<L>() && (KM & ((1u << kAC) | (1u << kAP))))     ? BP_MINB_I15
                                                                                                 : BP_MINB1)
k_exact_fast(const __grid_constant__ ExactArgs<L> a, double2* __restrict__ unit_out,
             unsigned long long* __restrict__ hist, const ExactArgs<L>* __restrict__ ga,
             unsigned long long* __restrict__ work) {
  // ga: the device copy of the argument block followed by the shared-memory
  // image (below); the leaf loops read the parameter bank (uniform loads).
  constexpr bool kAC_ = (KM >> kAC) & 1, kAP_ = (KM >> kAP) & 1, kFL_ = (KM >> kFL) & 1,
                 kFLP_ = (KM >> kFLP) & 1;
  // table slots in kind order AC, AP, FL, FLP
  constexpr int NT = (int)kAC_ + (int)kAP_ + (int)kFL_ + (int)kFLP_;
  static_assert(NT <= 2, "at most two tables per launch");
  static_assert(!(kAC_ && kAP_), "the Asian call and put share one threshold slot order; launch them apart");

  __shared__ unsigned long long shist[kMaxN + 2];
  static_assert(BP_GRAY && BP_FOLD, "K1 runs the Gray-code fold leaf block");
  // The shared tables as ONE image (k1_smem_layout, dynamic shared memory):
  // the weights (zero padded), the lookback kinds' W1/W2, the Gray tables of
  // the classes the screen leaves to fp64 compares, and per screened slot the
  // I15 entry tables, screened values and tie-run ends.  The host builds the
  // image once per lattice after the argument block (ga, device memory);
  // every CTA copies it with 16-byte loads.  After the image come the class
  // prefix sums the exact walk reads (global memory).
  constexpr K1SmemLayout LY = k1_smem_layout<L>(KM);
  static_assert(kGraySlots == 64, "k1_smem_layout assumes 64 Gray slots per group");
  extern __shared__ __align__(16) unsigned char simg[];
  const char* gimg = reinterpret_cast<const char*>(ga) + align16(sizeof(ExactArgs<L>));
  const double* gcpre = reinterpret_cast<const double*>(gimg + LY.total);
  {
    const uint4* src = reinterpret_cast<const uint4*>(gimg);
    uint4* dst = reinterpret_cast<uint4*>(simg);
    // every load of the thread issued before the first store (one memory latency)
    constexpr int n16 = (int)(LY.total / 16), per = (n16 + 255) / 256;
    uint4 v[per];
#pragma unroll
    for (int r = 0; r < per; ++r) {
      const int i = threadIdx.x + 256 * r;
      if (i < n16) v[r] = __ldg(src + i);
    }
#pragma unroll
    for (int r = 0; r < per; ++r) {
      const int i = threadIdx.x + 256 * r;
      if (i < n16) dst[i] = v[r];
    }
  }
  // nibble tables of the prefix walk: 4 steps with up pattern nb (first step = bit 3)
  __shared__ double4 snib[16];
  if (threadIdx.x < 16) {
    double r = 1.0, c = 0.0, mx = 0.0, mn = __longlong_as_double(0x7ff0000000000000ll);
    for (int l = 0; l < 4; ++l) {
      r *= ((threadIdx.x >> (3 - l)) & 1) ? a.s.u : a.s.d;
      c += r;
      mx = fmax(mx, r);
      mn = fmin(mn, r);
    }
    snib[threadIdx.x] = make_double4(r, c, mx, mn);
  }
  if (CNT)
    for (int i = threadIdx.x; i < kMaxN + 2; i += blockDim.x) shist[i] = 0ull;
  __syncthreads();

  const int lane = threadIdx.x & 31;
  const unsigned long long warp_global = (blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x) >> 5;
  const unsigned long long n_warps = (gridDim.x * (unsigned long long)blockDim.x) >> 5;
  unsigned long long leaves = 0, code_sum = 0;
  const ExactScalars& sc = a.s;
  constexpr bool kSplit = BP_SLOT_MAJOR && NT == 2;
  // virtual units: [0, U) the launch's units; slot-major, [0, U) are slot 0's
  // kinds (and the class-closed European kinds, and the bookkeeping) and
  // [U, 2U) slot 1's kind
  constexpr unsigned K1 = kSplit ? second_table_bit(KM) : 0u, K0 = KM & ~K1;
  const unsigned long long U = sc.unit_end - sc.unit_first, total = kSplit ? 2 * U : U;
  unsigned long long v = warp_global;
  while (v < total) {
    // the next unit's index is requested now and read after this unit
    unsigned long long next = v + n_warps;
    if (BP_K1_DYNAMIC && lane == 0) next = n_warps + atomicAdd(work, 1ull);
    if constexpr (kSplit) {
      if (v < U)
        fast_unit<L, KM, K0, CNT>(a, snib, simg, gcpre, sc.unit_first + v, lane, unit_out, shist, leaves, code_sum);
      else
        fast_unit<L, KM, K1, false>(a, snib, simg, gcpre, sc.unit_first + (v - U), lane, unit_out, shist, leaves,
                                    code_sum);
    } else {
      fast_unit<L, KM, KM, CNT>(a, snib, simg, gcpre, sc.unit_first + v, lane, unit_out, shist, leaves, code_sum);
    }
    v = BP_K1_DYNAMIC ? __shfl_sync(0xffffffffu, next, 0) : next;
  }
  if (CNT) {
    atomicAdd(&hist[64], leaves);
    atomicAdd(&hist[65], code_sum);
    __syncthreads();
    for (int i = threadIdx.x; i < kMaxN + 1; i += blockDim.x)
      if (shist[i]) atomicAdd(&hist[i], shist[i]);
  }
}

// the dynamic shared-memory size of both instantiations (once per process
// and device; beyond 48 KB it must be opted into)
template <int L, unsigned KM>
void fast_smem_attr() {
  static bool done[64] = {false};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64 || done[dev]) return;
  constexpr int smem = (int)k1_smem_layout<L>(KM).total;
  cudaFuncSetAttribute(k_exact_fast<L, KM, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k_exact_fast<L, KM, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  done[dev] = true;
}

// launch wrappers
template <int L, unsigned KM>
cudaError_t launch_fast_t(const void* args, bool cnt, int grid, cudaStream_t st, double2* unit_out,
                          unsigned long long* hist, const void* dev_args, unsigned long long* work) {
  const ExactArgs<L>& a = *static_cast<const ExactArgs<L>*>(args);
  const ExactArgs<L>* ga = static_cast<const ExactArgs<L>*>(dev_args);
  if (!ga || !work) return cudaErrorInvalidValue;  // K1 needs its device image and unit counter
  constexpr size_t smem = k1_smem_layout<L>(KM).total;
  fast_smem_attr<L, KM>();
  if (cnt)
    k_exact_fast<L, KM, true><<<grid, 256, smem, st>>>(a, unit_out, hist, ga, work);
  else
    k_exact_fast<L, KM, false><<<grid, 256, smem, st>>>(a, unit_out, hist, ga, work);
  return cudaGetLastError();
}

template <int L, unsigned KM>
int occupancy_fast_t(bool cnt) {
  int n = 0;
  constexpr size_t smem = k1_smem_layout<L>(KM).total;
  fast_smem_attr<L, KM>();
  if (cnt)
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k_exact_fast<L, KM, true>, 256, smem);
  else
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k_exact_fast<L, KM, false>, 256, smem);
  return n;
}

}  // namespace bp

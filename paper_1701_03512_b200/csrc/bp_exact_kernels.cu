// Exact-enumeration kernels (K1 fast affine-threshold walk, K0 per-path walk,
// K2 super-block reduce, K6 leaf bookkeeping).  See bp_exact.cuh for the
// index decomposition and the math; reference: pkg/src/binpaths/exact.py:83-133.
#include <cmath>
#include "bp_exact.cuh"
#include "bp_kernels.h"

namespace bp {

__device__ __forceinline__ double u32_to_double(unsigned x) {
  // exact: 2^52 + x - 2^52
  return __hiloint2double(0x43300000, (int)x) - 4503599627370496.0;
}

// ---------------------------------------------------------------------------
// K1: affine-threshold enumeration.  KM = compile-time kind mask.
template <int L, unsigned KM, bool CNT>
__global__ void __launch_bounds__(256)
k_exact_fast(const __grid_constant__ ExactArgs<L> a, double2* __restrict__ unit_out,
             unsigned long long* __restrict__ hist) {
  constexpr int NL = 1 << L;
  constexpr int NC = L + 1;
  constexpr bool kAC_ = (KM >> kAC) & 1, kAP_ = (KM >> kAP) & 1, kFL_ = (KM >> kFL) & 1,
                 kFLP_ = (KM >> kFLP) & 1, kEC_ = (KM >> kEC) & 1, kEP_ = (KM >> kEP) & 1;
  constexpr bool needMx = kFL_, needMn = kFLP_;

  constexpr int NT_ = (int)(kAC_ || kAP_) + (int)kFL_ + (int)kFLP_;
  __shared__ double sw[kMaxN + 2 + NC];
  __shared__ unsigned long long shist[kMaxN + 2];
  // two-table kernels read the interleaved tables from shared memory (one
  // broadcast LDS.128 per leaf); one-table kernels read the constant bank
  __shared__ __align__(16) double stab[NT_ == 2 ? (2 << L) : 2];
  if (NT_ == 2)
    for (int i = threadIdx.x; i < (2 << L); i += blockDim.x) stab[i] = a.tab[i];
  for (int i = threadIdx.x; i < kMaxN + 2 + NC; i += blockDim.x) sw[i] = (i < kMaxN + 2) ? a.w[i] : 0.0;
  if (CNT)
    for (int i = threadIdx.x; i < kMaxN + 2; i += blockDim.x) shist[i] = 0ull;
  __syncthreads();

  const ExactScalars& sc = a.s;
  const int lane = threadIdx.x & 31;
  const unsigned long long warp_global = (blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x) >> 5;
  const unsigned long long n_warps = (gridDim.x * (unsigned long long)blockDim.x) >> 5;
  const int zlo = lane & sc.zero;
  const double INF = __longlong_as_double(0x7ff0000000000000ll);
  unsigned long long leaves = 0, code_sum = 0;

  for (unsigned long long unit = sc.unit_first + warp_global; unit < sc.unit_end; unit += n_warps) {
    double ts[kNumKinds], tc[kNumKinds];
#pragma unroll
    for (int k = 0; k < kNumKinds; ++k) { ts[k] = 0.0; tc[k] = 0.0; }
   for (unsigned long long rr = 0; rr < (1ull << sc.q); ++rr) {
    const unsigned long long tp = (((unit << sc.q) | rr) << 5) | (unsigned long long)lane;  // thread prefix, Dp bits
    // --- prefix walk: steps 1..Dp (reference asset_path, model.py:164-172)
    double S = sc.S0, Sig = 0.0, Mx = 0.0, Mn = INF;
    int h = 0;
    for (int t = sc.Dp - 1; t >= 0; --t) {
      const int b = (int)((tp >> t) & 1ull);
      S *= b ? sc.u : sc.d;
      Sig += S;
      if (needMx) Mx = fmax(Mx, S);
      if (needMn) Mn = fmin(Mn, S);
      h += b;
    }

    for (int j = 0; j < sc.n_mid; ++j) {
      // --- node state at depth D
      const double Sn = S * a.mid_e[j];
      const double Sg = fma(S, a.mid_c[j], Sig);
      const double Mxn = needMx ? fmax(Mx, S * a.mid_mx[j]) : 0.0;
      const double Mnn = needMn ? fmin(Mn, S * a.mid_mn[j]) : 0.0;
      const int hn = h + a.mid_h[j];
      const double base = Sg - sc.NK;
      // thresholds on the scaled tables
      double thC = 0.0, thX = 0.0, thN = 0.0;
      if (kAC_ || kAP_) thC = (-base / Sn) * sc.sc_up[0];
      if (kFL_) thX = (Mxn / Sn) * sc.sc_up[1];
      if (kFLP_) thN = (fmin(Mnn, sc.K) / Sn) * sc.sc_up[2];

      // --- the leaf block: 2^L leaves, one compare + one masked FMA each
      double accC[NC], accP[NC], accX[NC], accN[NC];
      unsigned cntC[NC], cntP[NC], cntX[NC], cntN[NC];
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        accC[c] = accP[c] = accX[c] = accN[c] = 0.0;
        cntC[c] = cntP[c] = cntX[c] = cntN[c] = 0u;
      }
      const int off = j & sc.zero;  // 0, opaque to the compiler
      constexpr int NT = (int)(kAC_ || kAP_) + (int)kFL_ + (int)kFLP_;  // tables in use (<= 2)
      const double2* tb = reinterpret_cast<const double2*>(NT == 2 ? stab : a.tab) + off;
#pragma unroll
      for (int s2 = 0; s2 < NL / 2; ++s2) {
        // NT == 1: one double2 = leaves (2 s2, 2 s2 + 1) of the single table
        // NT == 2: two double2 = (first, second) table values of the two leaves
        double2 va = make_double2(0.0, 0.0), vb = make_double2(0.0, 0.0);
        if (NT == 1) va = tb[s2];
        if (NT == 2) { va = tb[2 * s2]; vb = tb[2 * s2 + 1]; }
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          const int s = 2 * s2 + hh;
          const int cls = __popc(s);
          const double x0 = (NT == 1) ? (hh ? va.y : va.x) : (hh ? vb.x : va.x);
          const double x1 = (NT == 1) ? 0.0 : (hh ? vb.y : va.y);
          if (kAC_ || kAP_) {
            const double c = x0;
            if (kAC_) {
              const unsigned mh = (c > thC) ? kMaskHi : 0u;
              accC[cls] = fma(__hiloint2double((int)mh, zlo), c, accC[cls]);
              cntC[cls] += mh;
            }
            if (kAP_) {
              const unsigned mh = (c < thC) ? kMaskHi : 0u;
              accP[cls] = fma(__hiloint2double((int)mh, zlo), c, accP[cls]);
              cntP[cls] += mh;
            }
          }
          if (kFL_) {
            const double c = (kAC_ || kAP_) ? x1 : x0;
            const unsigned mh = (c > thX) ? kMaskHi : 0u;
            accX[cls] = fma(__hiloint2double((int)mh, zlo), c, accX[cls]);
            cntX[cls] += mh;
          }
          if (kFLP_) {
            const double c = (kAC_ || kAP_ || kFL_) ? x1 : x0;
            const unsigned mh = (c < thN) ? kMaskHi : 0u;
            accN[cls] = fma(__hiloint2double((int)mh, zlo), c, accN[cls]);
            cntN[cls] += mh;
          }
        }
      }
      // --- class finalisation: node value = sum_c w[h+c] * contrib_c
      double vAC = 0.0, vAP = 0.0, vFL = 0.0, vFLP = 0.0, vEC = 0.0, vEP = 0.0;
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        const double wv = sw[hn + c];
        const double bc = a.b_cls[c];
        if (kAC_) {
          const double A = accC[c] * sc.sc_dn[0];
          const double n = u32_to_double(cntC[c] >> 24);
          vAC = fma(wv, fma(Sn, A, base * n), vAC);
        }
        if (kAP_) {
          const double A = accP[c] * sc.sc_dn[0];
          const double n = u32_to_double(cntP[c] >> 24);
          vAP = fma(wv, fma(-Sn, A, -base * n), vAP);
        }
        if (kFL_) {
          const double A = accX[c] * sc.sc_dn[1];
          const double n = u32_to_double(cntX[c] >> 24);
          // S A + Mx (C_c - n) - S e_c C_c
          const double t = fma(Sn, A, Mxn * (bc - n));
          vFL = fma(wv, fma(-Sn * a.e_cls[c], bc, t), vFL);
        }
        if (kFLP_) {
          const double A = accN[c] * sc.sc_dn[2];
          const double n = u32_to_double(cntN[c] >> 24);
          const double flat = fmax(sc.K - Mnn, 0.0);
          const double t = fma(sc.K, n, -Sn * A);
          vFLP = fma(wv, fma(bc - n, flat, t), vFLP);
        }
        if (kEC_) vEC = fma(wv, bc * fmax(fma(Sn, a.e_cls[c], -sc.K), 0.0), vEC);
        if (kEP_) vEP = fma(wv, bc * fmax(fma(-Sn, a.e_cls[c], sc.K), 0.0), vEP);
      }
      if (kAC_) comp_add(ts[kAC], tc[kAC], vAC);
      if (kAP_) comp_add(ts[kAP], tc[kAP], vAP);
      if (kFL_) comp_add(ts[kFL], tc[kFL], vFL);
      if (kFLP_) comp_add(ts[kFLP], tc[kFLP], vFLP);
      if (kEC_) comp_add(ts[kEC], tc[kEC], vEC);
      if (kEP_) comp_add(ts[kEP], tc[kEP], vEP);

      if (CNT) {
        // leaf bookkeeping (K6): leaves per total up count, code coverage
        const unsigned long long node = (tp << sc.m) | (unsigned long long)j;
#pragma unroll
        for (int c = 0; c < NC; ++c) atomicAdd(&shist[hn + c], (unsigned long long)a.b_cls[c]);
        leaves += (unsigned long long)NL;
        // sum of codes node*2^L + s, s < 2^L
        code_sum += (node << (2 * L)) + (((unsigned long long)NL * (NL - 1)) >> 1);
      }
    }
   }  // rr
    // --- per-unit partial: fixed warp tree, lane 0 stores
#pragma unroll
    for (int k = 0; k < kNumKinds; ++k) {
      if (!((KM >> k) & 1)) continue;
      double s = ts[k], c = tc[k];
      warp_comp_reduce(s, c);
      if (lane == 0) unit_out[unit * kNumKinds + k] = make_double2(s, c);
    }
  }
  if (CNT) {
    atomicAdd(&hist[64], leaves);
    atomicAdd(&hist[65], code_sum);
    __syncthreads();
    for (int i = threadIdx.x; i < kMaxN + 1; i += blockDim.x)
      if (shist[i]) atomicAdd(&hist[i], shist[i]);
  }
}

// ---------------------------------------------------------------------------
// K0: per-path walk (any per-step probabilities).  Lane owns 2^g codes.
template <bool CNT>
__global__ void __launch_bounds__(256)
k_exact_generic(const __grid_constant__ GenericArgs a, double2* __restrict__ unit_out,
                unsigned long long* __restrict__ hist) {
  __shared__ unsigned long long shist[kMaxN + 2];
  if (CNT) {
    for (int i = threadIdx.x; i < kMaxN + 2; i += blockDim.x) shist[i] = 0ull;
    __syncthreads();
  }
  const int lane = threadIdx.x & 31;
  const unsigned long long warp_global = (blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x) >> 5;
  const unsigned long long n_warps = (gridDim.x * (unsigned long long)blockDim.x) >> 5;
  const double INF = __longlong_as_double(0x7ff0000000000000ll);
  unsigned long long leaves = 0, code_sum = 0;
  for (unsigned long long unit = a.unit_first + warp_global; unit < a.unit_end; unit += n_warps) {
    double ts[kNumKinds], tc[kNumKinds];
#pragma unroll
    for (int k = 0; k < kNumKinds; ++k) { ts[k] = 0.0; tc[k] = 0.0; }
    const unsigned long long c0 = ((unit << 5) | (unsigned long long)lane) << a.g;
    const unsigned long long cn = 1ull << a.g;
    for (unsigned long long i = 0; i < cn; ++i) {
      const unsigned long long code = c0 + i;
      if (code >= a.n_codes) break;
      double S = a.S0, Sig = 0.0, Mx = -INF, Mn = INF, w = 1.0;
      int h = 0;
      for (int t = a.N - 1; t >= 0; --t) {
        const int b = (int)((code >> t) & 1ull);
        const double p = a.p[a.N - 1 - t];
        w *= b ? p : 1.0 - p;
        S *= b ? a.u : a.d;
        Sig += S;
        Mx = fmax(Mx, S);
        Mn = fmin(Mn, S);
        h += b;
      }
      const double mean = Sig / (double)a.N;  // numpy mean: sum / N (payoffs.py:105-106)
      const double v[kNumKinds] = {fmax(S - a.K, 0.0), fmax(a.K - S, 0.0), fmax(a.K - mean, 0.0),
                                   fmax(a.K - Mn, 0.0), fmax(mean - a.K, 0.0), Mx - S};
#pragma unroll
      for (int k = 0; k < kNumKinds; ++k)
        if ((a.kinds >> k) & 1) comp_add(ts[k], tc[k], w * v[k]);
      if (CNT) {
        atomicAdd(&shist[h], 1ull);
        leaves += 1;
        code_sum += code;
      }
    }
#pragma unroll
    for (int k = 0; k < kNumKinds; ++k) {
      if (!((a.kinds >> k) & 1)) continue;
      double s = ts[k] * a.disc, c = tc[k] * a.disc;
      warp_comp_reduce(s, c);
      if (lane == 0) unit_out[unit * kNumKinds + k] = make_double2(s, c);
    }
  }
  if (CNT) {
    atomicAdd(&hist[64], leaves);
    atomicAdd(&hist[65], code_sum);
    __syncthreads();
    for (int i = threadIdx.x; i < kMaxN + 1; i += blockDim.x)
      if (shist[i]) atomicAdd(&hist[i], shist[i]);
  }
}

// ---------------------------------------------------------------------------
// K2: super-block reduce.  Block b reduces the units of super-block
// sb_first + b in a fixed order (thread-contiguous chunks, fixed tree), and
// writes (sum, comp) per kind scaled by scale[k] (1/N for Asian kinds).
__global__ void __launch_bounds__(256)
k_sb_reduce(const double2* __restrict__ unit_out, unsigned long long units_per_sb, int sb_first,
            unsigned kinds, double scale_asian, double* __restrict__ out) {
  __shared__ double ss[256], sc2[256];
  const unsigned long long u0 = (unsigned long long)(sb_first + blockIdx.x) * units_per_sb;
  for (int k = 0; k < kNumKinds; ++k) {
    if (!((kinds >> k) & 1)) continue;
    double s = 0.0, c = 0.0;
    const unsigned long long per = (units_per_sb + blockDim.x - 1) / blockDim.x;
    const unsigned long long lo = threadIdx.x * per;
    const unsigned long long hi = lo + per < units_per_sb ? lo + per : units_per_sb;
    for (unsigned long long u = lo; u < hi; ++u) {
      const double2 v = unit_out[(u0 + u) * kNumKinds + k];
      comp_merge(s, c, v.x, v.y);
    }
    ss[threadIdx.x] = s;
    sc2[threadIdx.x] = c;
    __syncthreads();
    for (int stride = blockDim.x / 2; stride > 0; stride >>= 1) {
      if (threadIdx.x < stride) {
        double a_s = ss[threadIdx.x], a_c = sc2[threadIdx.x];
        comp_merge(a_s, a_c, ss[threadIdx.x + stride], sc2[threadIdx.x + stride]);
        ss[threadIdx.x] = a_s;
        sc2[threadIdx.x] = a_c;
      }
      __syncthreads();
    }
    if (threadIdx.x == 0) {
      const double f = (k == kAC || k == kAP) ? scale_asian : 1.0;
      out[(blockIdx.x * kNumKinds + k) * 2 + 0] = ss[0] * f;
      out[(blockIdx.x * kNumKinds + k) * 2 + 1] = sc2[0] * f;
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// launch wrappers
template <int L, unsigned KM>
static cudaError_t launch_fast_t(const void* args, bool cnt, int grid, cudaStream_t st, double2* unit_out,
                                 unsigned long long* hist) {
  const ExactArgs<L>& a = *static_cast<const ExactArgs<L>*>(args);
  if (cnt)
    k_exact_fast<L, KM, true><<<grid, 256, 0, st>>>(a, unit_out, hist);
  else
    k_exact_fast<L, KM, false><<<grid, 256, 0, st>>>(a, unit_out, hist);
  return cudaGetLastError();
}

template <int L, unsigned KM>
static int occupancy_fast_t(bool cnt) {
  int n = 0;
  if (cnt)
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k_exact_fast<L, KM, true>, 256, 0);
  else
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k_exact_fast<L, KM, false>, 256, 0);
  return n;
}

#define BP_FAST_KMS(X, L)                                                      \
  X(L, (1u << kAC)) X(L, (1u << kAP)) X(L, (1u << kFL)) X(L, (1u << kFLP))     \
  X(L, (1u << kEC)) X(L, (1u << kEP)) X(L, ((1u << kAC) | (1u << kFL)))

bool fast_kind_mask_supported(unsigned km) {
  switch (km) {
    case (1u << kAC): case (1u << kAP): case (1u << kFL): case (1u << kFLP):
    case (1u << kEC): case (1u << kEP): case ((1u << kAC) | (1u << kFL)):
      return true;
    default:
      return false;
  }
}

cudaError_t launch_exact_fast(int L, unsigned km, const void* args, bool cnt, int grid, cudaStream_t st,
                              double2* unit_out, unsigned long long* hist) {
#define BP_CASE(LL, KMV) \
  if (L == LL && km == (KMV)) return launch_fast_t<LL, (KMV)>(args, cnt, grid, st, unit_out, hist);
  BP_FAST_KMS(BP_CASE, 8)
#undef BP_CASE
  return cudaErrorInvalidValue;
}

int occupancy_exact_fast(int L, unsigned km, bool cnt) {
#define BP_CASE(LL, KMV) \
  if (L == LL && km == (KMV)) return occupancy_fast_t<LL, (KMV)>(cnt);
  BP_FAST_KMS(BP_CASE, 8)
#undef BP_CASE
  return 0;
}

size_t exact_args_size(int L) {
  switch (L) {
    case 8: return sizeof(ExactArgs<8>);
    default: return 0;
  }
}

cudaError_t launch_exact_generic(const GenericArgs& a, bool cnt, int grid, cudaStream_t st, double2* unit_out,
                                 unsigned long long* hist) {
  if (cnt)
    k_exact_generic<true><<<grid, 256, 0, st>>>(a, unit_out, hist);
  else
    k_exact_generic<false><<<grid, 256, 0, st>>>(a, unit_out, hist);
  return cudaGetLastError();
}

int occupancy_exact_generic(bool cnt) {
  int n = 0;
  if (cnt)
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k_exact_generic<true>, 256, 0);
  else
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k_exact_generic<false>, 256, 0);
  return n;
}

cudaError_t launch_sb_reduce(const double2* unit_out, unsigned long long units_per_sb, int sb_first, int sb_count,
                             unsigned kinds, double scale_asian, double* out, cudaStream_t st) {
  k_sb_reduce<<<sb_count, 256, 0, st>>>(unit_out, units_per_sb, sb_first, kinds, scale_asian, out);
  return cudaGetLastError();
}

}  // namespace bp

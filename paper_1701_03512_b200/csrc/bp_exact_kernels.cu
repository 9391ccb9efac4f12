// Exact-enumeration kernels (K1 fast affine-threshold walk, K0 per-path walk,
// K2 super-block reduce, K6 leaf bookkeeping).  See bp_exact.cuh for the
// index decomposition and the math; reference: pkg/src/binpaths/exact.py:83-133.
#include <cmath>
#include "bp_exact.cuh"
#include "bp_kernels.h"
#include "bp_leaf.cuh"

namespace bp {


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
// sb_first + b in a fixed order -- thread t merges units t, t + 256, ... in
// ascending order, then a fixed warp shuffle tree (warp_comp_reduce), then
// warp 0 merges the 8 warp sums the same way -- and writes (sum, comp) per
// kind scaled by scale[k] (1/N for Asian kinds).  Kinds in zero_kinds
// (requested by no launch group of the valuation) are written as 0, so every
// output entry is written exactly once per step.
__global__ void __launch_bounds__(256)
k_sb_reduce(const double2* __restrict__ unit_out, unsigned long long units_per_sb, int sb_first,
            unsigned kinds, unsigned zero_kinds, double scale_asian, double* __restrict__ out,
            unsigned long long* __restrict__ work) {
  if (work && blockIdx.x == 0 && threadIdx.x == 0) *work = 0ull;  // the K1 before us is done with it
  __shared__ double ws[kNumKinds][8], wc[kNumKinds][8];
  const unsigned long long u0 = (unsigned long long)(sb_first + blockIdx.x) * units_per_sb;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x < 2 * kNumKinds && ((zero_kinds >> (threadIdx.x >> 1)) & 1))
    out[blockIdx.x * kNumKinds * 2 + threadIdx.x] = 0.0;
  // all of the thread's loads first (every kind), then the merges
#pragma unroll
  for (int k = 0; k < kNumKinds; ++k) {
    if (!((kinds >> k) & 1)) continue;
    double s = 0.0, c = 0.0;
    for (unsigned long long u = threadIdx.x; u < units_per_sb; u += blockDim.x) {
      const double2 v = unit_out[(u0 + u) * kNumKinds + k];
      comp_merge(s, c, v.x, v.y);
    }
    warp_comp_reduce(s, c);
    if (lane == 0) {
      ws[k][warp] = s;
      wc[k][warp] = c;
    }
  }
  __syncthreads();
  if (warp == 0) {
#pragma unroll
    for (int k = 0; k < kNumKinds; ++k) {
      if (!((kinds >> k) & 1)) continue;
      double s = lane < 8 ? ws[k][lane] : 0.0, c = lane < 8 ? wc[k][lane] : 0.0;
      warp_comp_reduce(s, c);
      if (lane == 0) {
        const double f = (k == kAC || k == kAP) ? scale_asian : 1.0;
        out[(blockIdx.x * kNumKinds + k) * 2 + 0] = s * f;
        out[(blockIdx.x * kNumKinds + k) * 2 + 1] = c * f;
      }
    }
  }
}

// ---------------------------------------------------------------------------
// K1 launchers: defined in bp_exact_fast.cuh, one explicit instantiation per
// (L, kind mask) in bp_exact_fast_inst.cu (compiled once per BP_FAST_PART).
template <int L, unsigned KM>
cudaError_t launch_fast_t(const void* args, bool cnt, int grid, cudaStream_t st, double2* unit_out,
                          unsigned long long* hist, const void* dev_args, unsigned long long* work);
template <int L, unsigned KM>
int occupancy_fast_t(bool cnt);



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
                              double2* unit_out, unsigned long long* hist, const void* dev_args,
                              unsigned long long* work) {
#define BP_CASE(LL, KMV) \
  if (L == LL && km == (KMV)) return launch_fast_t<LL, (KMV)>(args, cnt, grid, st, unit_out, hist, dev_args, work);
  BP_FAST_KMS(BP_CASE, 8)
  BP_FAST_KMS(BP_CASE, 9)
#undef BP_CASE
  return cudaErrorInvalidValue;
}

int occupancy_exact_fast(int L, unsigned km, bool cnt) {
#define BP_CASE(LL, KMV) \
  if (L == LL && km == (KMV)) return occupancy_fast_t<LL, (KMV)>(cnt);
  BP_FAST_KMS(BP_CASE, 8)
  BP_FAST_KMS(BP_CASE, 9)
#undef BP_CASE
  return 0;
}

size_t exact_args_size(int L) {
  switch (L) {
    case 8: return sizeof(ExactArgs<8>);
    case 9: return sizeof(ExactArgs<9>);
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
                             unsigned kinds, unsigned zero_kinds, double scale_asian, double* out, cudaStream_t st,
                             unsigned long long* work) {
  k_sb_reduce<<<sb_count, 256, 0, st>>>(unit_out, units_per_sb, sb_first, kinds, zero_kinds, scale_asian, out, work);
  return cudaGetLastError();
}

}  // namespace bp

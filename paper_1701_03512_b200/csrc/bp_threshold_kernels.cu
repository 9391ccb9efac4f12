// K8: threshold-search engine (reported as EFFECTIVE paths/s).
//
// Same decomposition and math as K1 (bp_exact.cuh), but a node's inner block
// of 2^LT leaves is NOT visited leaf by leaf.  Inside each up-count class the
// inner values are sorted in the compare direction, so the in-the-money
// leaves of a node are a prefix of the class: a binary search for the node's
// threshold gives their count n_c, and the class prefix sum P_c[n_c] gives
// their sum.  Cost per node is O(sum_c log C(LT, c)) instead of O(2^LT); the
// value is the same exact expectation (parity tests compare both engines).
// Tables (sorted class values + prefix sums, one set per kind) live in global
// memory and stay L2/L1 resident.
#include "bp_kernels.h"
#include "bp_threshold.h"

namespace bp {

// number of entries > th (GT) or < th (!GT) in the sorted range v[0, n)
template <bool GT>
__device__ __forceinline__ int count_itm(const double* __restrict__ v, int n, double th) {
  int lo = 0, hi = n;  // invariant: the ITM entries are exactly v[0, lo) once lo == hi
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    const double x = __ldg(&v[mid]);
    const bool itm = GT ? (x > th) : (x < th);
    if (itm) lo = mid + 1; else hi = mid;
  }
  return lo;
}

__global__ void __launch_bounds__(256)
k_exact_threshold(const __grid_constant__ ThresholdArgs a, double2* __restrict__ unit_out) {
  const int lane = threadIdx.x & 31;
  const unsigned long long warp_global = (blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x) >> 5;
  const unsigned long long n_warps = (gridDim.x * (unsigned long long)blockDim.x) >> 5;
  const double INF = __longlong_as_double(0x7ff0000000000000ll);
  const int NC = a.LT + 1;
  for (unsigned long long unit = a.unit_first + warp_global; unit < a.unit_end; unit += n_warps) {
    double ts[kNumKinds], tc[kNumKinds];
#pragma unroll
    for (int k = 0; k < kNumKinds; ++k) { ts[k] = 0.0; tc[k] = 0.0; }
    for (unsigned long long rr = 0; rr < (1ull << a.q); ++rr) {
      const unsigned long long tp = (((unit << a.q) | rr) << 5) | (unsigned long long)lane;
      for (unsigned long long j = 0; j < (1ull << a.m); ++j) {
        const unsigned long long node = (tp << a.m) | j;
        double S = a.S0, Sig = 0.0, Mx = 0.0, Mn = INF;
        int h = 0;
        for (int t = a.D - 1; t >= 0; --t) {
          const int b = (int)((node >> t) & 1ull);
          S *= b ? a.u : a.d;
          Sig += S;
          Mx = fmax(Mx, S);
          Mn = fmin(Mn, S);
          h += b;
        }
        const double base = Sig - a.NK;
        const double rS = 1.0 / S;
        int slot = 0;
#pragma unroll
        for (int k = 0; k < kNumKinds; ++k) {
          if (!((a.kinds >> k) & 1)) continue;
          double v = 0.0;
          if (k == kEC || k == kEP) {
            for (int c = 0; c < NC; ++c) {
              const double bc = a.b_cls[c];
              const double term = (k == kEC) ? fmax(fma(S, a.e_cls[c], -a.K), 0.0)
                                             : fmax(fma(-S, a.e_cls[c], a.K), 0.0);
              v = fma(a.w[h + c], bc * term, v);
            }
          } else {
            const bool gt = (k == kAC || k == kFL);
            const double th = (k == kAC || k == kAP) ? -base * rS : (k == kFL) ? Mx * rS : fmin(Mn, a.K) * rS;
            const double* vals = a.val[slot];
            const double* pre = a.pre[slot];
            ++slot;
            for (int c = 0; c < NC; ++c) {
              const int off = a.class_off[c], len = a.class_off[c + 1] - off;
              const int n = gt ? count_itm<true>(vals + off, len, th) : count_itm<false>(vals + off, len, th);
              const double A = __ldg(&pre[off + c + n]);  // prefix sums carry one extra slot per class
              const double nd = (double)n, bc = a.b_cls[c];
              double contrib;
              if (k == kAC) contrib = fma(S, A, base * nd);
              else if (k == kAP) contrib = fma(-S, A, -base * nd);
              else if (k == kFL) contrib = fma(-S * a.e_cls[c], bc, fma(S, A, Mx * (bc - nd)));
              else contrib = fma(bc - nd, fmax(a.K - Mn, 0.0), fma(a.K, nd, -S * A));
              v = fma(a.w[h + c], contrib, v);
            }
          }
          comp_add(ts[k], tc[k], v);
        }
      }
    }
#pragma unroll
    for (int k = 0; k < kNumKinds; ++k) {
      if (!((a.kinds >> k) & 1)) continue;
      double s = ts[k], c = tc[k];
      warp_comp_reduce(s, c);
      if (lane == 0) unit_out[unit * kNumKinds + k] = make_double2(s, c);
    }
  }
}

cudaError_t launch_exact_threshold(const ThresholdArgs& a, int grid, cudaStream_t st, double2* unit_out) {
  k_exact_threshold<<<grid, 256, 0, st>>>(a, unit_out);
  return cudaGetLastError();
}

int occupancy_exact_threshold() {
  int n = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k_exact_threshold, 256, 0);
  return n;
}

}  // namespace bp

// K3: batched exact pricing -- many independent trees (same N), one payoff.
//
// The reference has no batch API; its callers loop value_exact_parallel over
// requests (exact.py:112-133).  Here one CTA group owns one option: the CTA
// builds that option's inner / middle tables and weights in shared memory
// (each option has its own u, d, p), then runs the same affine-threshold
// leaf block as K1 (bp_exact_kernels.cu) with the tables read from shared
// memory (broadcast LDS), and reduces its partial in a fixed order.
#include <cmath>
#include "bp_kernels.h"

namespace bp {

constexpr int kBL = 8;             // inner bits
constexpr int kBM = 6;             // middle bits
constexpr int kBThreads = 256;

struct BatchArgs {
  int N;
  unsigned kind;
  int cpo_log2;  // CTAs per option = 2^cpo_log2
};

__device__ __forceinline__ double bu32_to_double(unsigned x) {
  return __hiloint2double(0x43300000, (int)x) - 4503599627370496.0;
}

template <unsigned KIND>
__global__ void __launch_bounds__(kBThreads)
k_exact_batch(const BatchOption* __restrict__ opts, BatchArgs ba, double2* __restrict__ partial) {
  constexpr int NL = 1 << kBL, NC = kBL + 1, NMID = 1 << kBM;
  constexpr bool AC = KIND == kAC, AP = KIND == kAP, FL = KIND == kFL, FLP = KIND == kFLP, EC = KIND == kEC,
                 EP = KIND == kEP;
  constexpr bool TAB = AC || AP || FL || FLP;
  __shared__ __align__(16) double tab[NL];
  __shared__ double mid_c[NMID], mid_e[NMID], mid_x[NMID];
  __shared__ int mid_h[NMID];
  __shared__ double w[kMaxN + 2 + NC];
  __shared__ double e_cls[NC], b_cls[NC];
  __shared__ double s_up, s_dn;
  __shared__ double red_s[kBThreads], red_c[kBThreads];

  const int opt = blockIdx.x >> ba.cpo_log2;
  const int part = blockIdx.x & ((1 << ba.cpo_log2) - 1);
  const BatchOption o = opts[opt];
  const int N = ba.N, D = N - kBL, Dp = D - kBM;
  const int tid = threadIdx.x;

  // ---- per-option tables (the walk of csrc/bp_capi.cu build_inner)
  for (int s = tid; s < NL; s += kBThreads) {
    double r = 1.0, c = 0.0, mx = 0.0, mn = INFINITY;
    for (int j = 0; j < kBL; ++j) {
      r *= ((s >> (kBL - 1 - j)) & 1) ? o.u : o.d;
      c += r;
      mx = fmax(mx, r);
      mn = fmin(mn, r);
    }
    tab[s] = (AC || AP) ? c : FL ? mx : mn;
  }
  for (int j = tid; j < NMID; j += kBThreads) {
    double r = 1.0, c = 0.0, mx = 0.0, mn = INFINITY;
    int h = 0;
    for (int t = 0; t < kBM; ++t) {
      const int b = (j >> (kBM - 1 - t)) & 1;
      r *= b ? o.u : o.d;
      c += r;
      mx = fmax(mx, r);
      mn = fmin(mn, r);
      h += b;
    }
    mid_c[j] = c;
    mid_e[j] = r;
    mid_x[j] = FL ? mx : mn;
    mid_h[j] = h;
  }
  for (int h = tid; h < kMaxN + 2 + NC; h += kBThreads)
    w[h] = (h <= N) ? o.disc * pow(o.p, (double)h) * pow(1.0 - o.p, (double)(N - h)) : 0.0;
  if (tid < NC) {
    double r = 1.0, b = 1.0;
    for (int j = 0; j < tid; ++j) r *= o.u;
    for (int j = tid; j < kBL; ++j) r *= o.d;
    for (int j = 0; j < tid; ++j) b = b * (kBL - j) / (j + 1);
    e_cls[tid] = r;
    b_cls[tid] = rint(b);
  }
  __syncthreads();
  if (tid == 0) {
    // tables are increasing in every up bit when u > d: the minimum is entry 0
    int e = 0;
    frexp(tab[0], &e);
    s_up = ldexp(1.0, 1 - e);
    s_dn = ldexp(1.0, kMaskExp - (1 - e));
  }
  __syncthreads();
  for (int s = tid; s < NL; s += kBThreads) tab[s] *= s_up;
  __syncthreads();

  const double NK = (double)N * o.K;
  const int zlo = tid & (ba.N >> 10);  // 0 (N < 1024), opaque to the compiler
  const double INF = __longlong_as_double(0x7ff0000000000000ll);
  double ts = 0.0, tc = 0.0;
  const unsigned long long n_pre = 1ull << Dp;
  const unsigned long long per = n_pre >> ba.cpo_log2;
  const unsigned long long p0 = (unsigned long long)part * per;
  for (unsigned long long pi = p0 + tid; pi < p0 + per; pi += kBThreads) {
    double S = o.S0, Sig = 0.0, X = FL ? 0.0 : INF;
    int h = 0;
    for (int t = Dp - 1; t >= 0; --t) {
      const int b = (int)((pi >> t) & 1ull);
      S *= b ? o.u : o.d;
      Sig += S;
      if (FL) X = fmax(X, S);
      if (FLP) X = fmin(X, S);
      h += b;
    }
    for (int j = 0; j < NMID; ++j) {
      const double Sn = S * mid_e[j];
      const double Sg = fma(S, mid_c[j], Sig);
      const double Xn = FL ? fmax(X, S * mid_x[j]) : FLP ? fmin(X, S * mid_x[j]) : 0.0;
      const int hn = h + mid_h[j];
      const double base = Sg - NK;
      double th = 0.0;
      if (AC || AP) th = (-base / Sn) * s_up;
      if (FL) th = (Xn / Sn) * s_up;
      if (FLP) th = (fmin(Xn, o.K) / Sn) * s_up;
      double acc[NC];
      unsigned cnt[NC];
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        acc[c] = 0.0;
        cnt[c] = 0u;
      }
      if (TAB) {
        const double2* tb = reinterpret_cast<const double2*>(tab) + (j & zlo);
#pragma unroll
        for (int s2 = 0; s2 < NL / 2; ++s2) {
          const double2 v = tb[s2];
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) {
            const int s = 2 * s2 + hh;
            const int cls = __popc(s);
            const double c = hh ? v.y : v.x;
            const bool itm = (AC || FL) ? (c > th) : (c < th);
            const unsigned mh = itm ? kMaskHi : 0u;
            acc[cls] = fma(__hiloint2double((int)mh, zlo), c, acc[cls]);
            cnt[cls] += mh;
          }
        }
      }
      double v = 0.0;
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        const double wv = w[hn + c];
        const double bc = b_cls[c];
        const double A = acc[c] * s_dn;
        const double n = bu32_to_double(cnt[c] >> 24);
        double contrib = 0.0;
        if (AC) contrib = fma(Sn, A, base * n);
        if (AP) contrib = fma(-Sn, A, -base * n);
        if (FL) contrib = fma(-Sn * e_cls[c], bc, fma(Sn, A, Xn * (bc - n)));
        if (FLP) contrib = fma(bc - n, fmax(o.K - Xn, 0.0), fma(o.K, n, -Sn * A));
        if (EC) contrib = bc * fmax(fma(Sn, e_cls[c], -o.K), 0.0);
        if (EP) contrib = bc * fmax(fma(-Sn, e_cls[c], o.K), 0.0);
        v = fma(wv, contrib, v);
      }
      comp_add(ts, tc, v);
    }
  }
  // fixed-order CTA reduce
  red_s[tid] = ts;
  red_c[tid] = tc;
  __syncthreads();
  for (int stride = kBThreads / 2; stride > 0; stride >>= 1) {
    if (tid < stride) {
      double a = red_s[tid], c = red_c[tid];
      comp_merge(a, c, red_s[tid + stride], red_c[tid + stride]);
      red_s[tid] = a;
      red_c[tid] = c;
    }
    __syncthreads();
  }
  if (tid == 0) {
    const double f = (AC || AP) ? 1.0 / N : 1.0;
    partial[blockIdx.x] = make_double2(red_s[0] * f, red_c[0] * f);
  }
}

__global__ void k_batch_combine(const double2* __restrict__ partial, int n_opts, int cpo_log2, double* __restrict__ values) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_opts) return;
  double s = 0.0, c = 0.0;
  for (int k = 0; k < (1 << cpo_log2); ++k) {
    const double2 p = partial[((long long)i << cpo_log2) + k];
    comp_merge(s, c, p.x, p.y);
  }
  values[i] = s + c;
}

int batch_ctas_per_option(int n_opts) {
  // enough CTAs to fill 148 SMs x 4 resident CTAs, at most 16 per option
  int l = 0;
  while (l < 4 && (long long)n_opts << l < 148 * 4) ++l;
  return l;
}

cudaError_t launch_exact_batch(const BatchOption* opts_dev, int n_opts, int N, unsigned kind, double* values_dev,
                               double2* scratch_dev, int cpo_log2, cudaStream_t st) {
  BatchArgs ba{N, kind, cpo_log2};
  const int grid = n_opts << cpo_log2;
#define BP_B_CASE(K) \
  case K: k_exact_batch<K><<<grid, kBThreads, 0, st>>>(opts_dev, ba, scratch_dev); break;
  switch (kind) {
    BP_B_CASE(kEC) BP_B_CASE(kEP) BP_B_CASE(kAP) BP_B_CASE(kFLP) BP_B_CASE(kAC) BP_B_CASE(kFL)
    default: return cudaErrorInvalidValue;
  }
#undef BP_B_CASE
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  k_batch_combine<<<(n_opts + 255) / 256, 256, 0, st>>>(scratch_dev, n_opts, cpo_log2, values_dev);
  return cudaGetLastError();
}

}  // namespace bp

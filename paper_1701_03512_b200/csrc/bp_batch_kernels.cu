// K3: batched exact pricing -- many independent trees (same N), one payoff.
//
// The reference has no batch API; its callers loop value_exact_parallel over
// requests (exact.py:112-133).  Here a group of CTAs owns one option: every
// CTA builds that option's tables in shared memory (each option has its own
// u, d, p) -- the inner table sorted inside each up-count class by a rank
// computation, the group prefix sums, the middle tables and the weights --
// and then runs the same explicit leaf block as K1 (bp_leaf.cuh: Gray-code
// predicate counting, each class folded into two per-node sums as it
// completes) over its share of the option's thread prefixes, nodes in pairs.
// Partials are reduced in a fixed order (CTA tree, then ascending CTA index
// per option).
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include "bp_kernels.h"
#include "bp_leaf.cuh"

namespace bp {

constexpr int kBL = 9;   // inner bits (as K1; the screen's per-class work amortizes over bigger classes)
constexpr int kBM = 6;   // middle bits
constexpr int kBThreads = 256;
constexpr int kBNP = 2;  // nodes per leaf block

struct BatchArgs {
  int N;
  unsigned kind;
  BatchLayout lay;
};

// Class layout of the inner block for a RUNTIME class index: binom() and
// class_start() are constexpr loops with 64-bit divisions; called with a
// runtime argument they ran on the device (6 % of K3's instructions).  One
// compile-time table instead.
struct BatchClassTab {
  int start[kBL + 2], size[kBL + 1];
  bool screened[kBL + 1];
  unsigned short cm[1 << kBL];  // class-major position of leaf s (ascending s inside a class)
  constexpr BatchClassTab() : start{}, size{}, screened{}, cm{} {
    int seen[kBL + 1] = {};
    for (int c = 0; c <= kBL; ++c) {
      start[c] = class_start(kBL, c);
      size[c] = binom(kBL, c);
      screened[c] = i15_class(kBL, c);
    }
    start[kBL + 1] = 1 << kBL;
    for (int s = 0; s < (1 << kBL); ++s) {
      int c = 0;
      for (int b = 0; b < kBL; ++b) c += (s >> b) & 1;
      cm[s] = (unsigned short)(start[c] + seen[c]++);
    }
  }
};
__constant__ BatchClassTab c_btab{};

// group prefix sums of class C (compile-time layout: no runtime binomials)
template <int C, bool SMALL_ONLY>
__device__ inline void batch_group_prefix(const double* __restrict__ tab, double* __restrict__ gpre) {
  if constexpr (C <= kBL) {
    if constexpr (!(SMALL_ONLY && i15_class(kBL, C))) {
      constexpr int ng = class_groups(kBL, C), g0 = group_base(kBL, C), size = binom(kBL, C);
      for (int gi = threadIdx.x; gi < ng * kGroupSlots; gi += blockDim.x) {
        const int gl = gi / kGroupSlots, n = gi % kGroupSlots;
        const int len = min(kGroup, size - kGroup * gl);
        const int i0 = class_start(kBL, C) + kGroup * gl;
        double s = 0.0, cc = 0.0;
        for (int k = 0; k < n && k < len; ++k) comp_add(s, cc, tab[i0 + k]);
        gpre[g0 * kGroupSlots + gi] = s + cc;
      }
    }
    batch_group_prefix<C + 1, SMALL_ONLY>(tab, gpre);
  }
}

template <unsigned KIND>
#ifndef BP_K3_MINB
#define BP_K3_MINB 3  // resident CTAs per SM targeted by K3
#endif
__global__ void __launch_bounds__(kBThreads, BP_K3_MINB)
k_exact_batch(const BatchOption* __restrict__ opts, BatchArgs ba, double2* __restrict__ partial) {
  constexpr int NL = 1 << kBL, NC = kBL + 1, NMID = 1 << kBM, NG = n_groups(kBL), NP = kBNP;
  constexpr bool AC = KIND == kAC, AP = KIND == kAP, FL = KIND == kFL, FLP = KIND == kFLP, EC = KIND == kEC,
                 EP = KIND == kEP;
  constexpr bool TAB = AC || AP || FL || FLP;
  constexpr bool DESC = AC || FL;  // compare direction '>' -> sort descending
  __shared__ __align__(16) double tab[NL];
  __shared__ double gpre[NG * kGroupSlots];
  // I15 screen (Asian kinds, as K1): the big classes' screen tables, built per
  // CTA from the option's sorted table; Gray tables only for the small classes
  constexpr bool I15 = (AC || AP) && i15_on<kBL>();
  constexpr int NGG = I15 ? n_small_groups<kBL>() : NG;
  __shared__ __align__(16) double2 sgray[TAB ? NGG * kGraySlots : 1];
  __shared__ float i15_s[I15 ? NC : 1], i15_o[I15 ? NC : 1];
  __shared__ double i15_cpre[I15 ? NL + NC : 1];
  __shared__ __align__(16) unsigned i15_xq[I15 ? NL : 4];
  __shared__ unsigned char i15_te[I15 ? NL : 4];
  __shared__ __align__(16) double2 i15_et[I15 ? 2 * i15_entries(kBL) : 1];
  __shared__ double sW1[(FL || FLP) ? kMaxN + 2 : 1], sW2[(FL || FLP) ? kMaxN + 2 : 1];
  __shared__ double mid_c[NMID], mid_e[NMID], mid_x[NMID];
  __shared__ int mid_h[NMID];
  __shared__ double w[kMaxN + 2 + NC];
  __shared__ double e_cls[NC], b_cls[NC];
  __shared__ double red_s[kBThreads / 32], red_c[kBThreads / 32];

  // CTA -> (option, part of 2^parts_log2): whole-layout options first, then the split tail
  const long long head = (long long)ba.lay.n_whole << ba.lay.base_log2;
  const bool in_head = (long long)blockIdx.x < head;
  const int parts_log2 = in_head ? ba.lay.base_log2 : ba.lay.tail_log2;
  const long long j = in_head ? (long long)blockIdx.x : (long long)blockIdx.x - head;
  const int opt = (in_head ? 0 : ba.lay.n_whole) + (int)(j >> parts_log2);
  const int part = (int)(j & ((1 << parts_log2) - 1));
  const BatchOption o = opts[opt];
  const int N = ba.N, D = N - kBL, Dp = D - kBM;
  const int tid = threadIdx.x;

  // ---- inner table: value of leaf s, then its position (class-major, sorted
  // in the compare direction inside the class; ties by leaf index)
  constexpr int PER = (NL + kBThreads - 1) / kBThreads;  // positions per thread
  double v[PER];
  int pos[PER], cmp[PER];
#pragma unroll
  for (int q = 0; q < PER; ++q) {
    const int sfx = tid + kBThreads * q;
    v[q] = 0.0;
    pos[q] = -1;
    cmp[q] = 0;
    if (TAB && sfx < NL) {
      double r = 1.0, c = 0.0, mx = 0.0, mn = INFINITY;
      for (int j = 0; j < kBL; ++j) {
        r *= ((sfx >> (kBL - 1 - j)) & 1) ? o.u : o.d;
        c += r;
        mx = fmax(mx, r);
        mn = fmin(mn, r);
      }
      v[q] = (AC || AP) ? c : FL ? mx : mn;
      cmp[q] = c_btab.cm[sfx];
      tab[cmp[q]] = v[q];  // staged class by class, leaf order inside a class
    }
  }
  __syncthreads();
#pragma unroll
  for (int q = 0; q < PER; ++q) {
    const int sfx = tid + kBThreads * q;
    if (TAB && sfx < NL) {
      const int cls = __popc(sfx);
      const int k0 = c_btab.start[cls], k1 = c_btab.start[cls + 1];
      int rank = 0;
      // the class's leaves only (a contiguous run of the staged table); ties
      // go by leaf index, which is the staged order: an equal value ahead of
      // this leaf counts, one behind it does not -- one compare per element
#pragma unroll 4
      for (int k = k0; k < cmp[q]; ++k) rank += DESC ? (tab[k] >= v[q]) : (tab[k] <= v[q]);
#pragma unroll 4
      for (int k = cmp[q] + 1; k < k1; ++k) rank += DESC ? (tab[k] > v[q]) : (tab[k] < v[q]);
      pos[q] = k0 + rank;
    }
  }
  __syncthreads();
#pragma unroll
  for (int q = 0; q < PER; ++q)
    if (pos[q] >= 0) tab[pos[q]] = v[q];
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
    double r = 1.0;
    for (int j = 0; j < tid; ++j) r *= o.u;
    for (int j = tid; j < kBL; ++j) r *= o.d;
    e_cls[tid] = r;
    b_cls[tid] = (double)c_btab.size[tid];
  }
  __syncthreads();
  // group prefix sums (compensated, rounded once), one (group, n) per thread;
  // the screened kinds need only the small classes' groups
  if (TAB) batch_group_prefix<0, I15>(tab, gpre);
  // lookback kinds: per node up count h, W1[h] = sum_c w[h+c] C(L,c) and
  // W2[h] = sum_c w[h+c] C(L,c) e_c (out-of-the-money and terminal terms)
  if (FL || FLP)
    for (int h = tid; h < kMaxN + 2; h += kBThreads) {
      double w1 = 0.0, w2 = 0.0;
      for (int c = 0; c < NC; ++c) {
        w1 = fma(w[h + c], b_cls[c], w1);
        w2 = fma(w[h + c] * b_cls[c], e_cls[c], w2);
      }
      sW1[h] = w1;
      sW2[h] = w2;
    }
  __syncthreads();
  // Gray-ordered {prefix sum, count} tables (count as a double: the fold form)
  if constexpr (I15) {
    gray_fill_small<kBL, 0>(reinterpret_cast<const double(*)[kGroupSlots]>(gpre), sgray);
    // per big class (one thread each): the monotone map onto [4, 32763] (as
    // the host builds it for K1, i15_layout) and the class prefix sums
    if (tid < NC && c_btab.screened[tid]) {
      const int c = tid, i0 = c_btab.start[c], len = c_btab.size[c];
      float lo = (float)tab[i0], hi = lo;
      for (int k = 0; k < len; ++k) {
        lo = fminf(lo, (float)tab[i0 + k]);
        hi = fmaxf(hi, (float)tab[i0 + k]);
      }
      const float range = hi - lo, amax = fmaxf(fabsf(lo), fabsf(hi));
      double sc = range > 0.0f ? 32759.0 / (double)range : 1.0;
      if (amax > 0.0f) sc = fmin(sc, 4194304.0 / (double)amax);
      if (!(sc > 0.0) || !isfinite(sc)) sc = 1.0;
      const float sf = (float)(DESC ? sc : -sc);
      const double off = (double)kI15Magic + 4.0 - (double)(DESC ? lo : hi) * (double)sf;
      i15_s[c] = sf;
      i15_o[c] = isfinite(off) ? (float)off : kI15Magic;
      double sum = 0.0, comp = 0.0;
      i15_cpre[i0 + c] = 0.0;
      for (int k = 0; k < len; ++k) {
        comp_add(sum, comp, tab[i0 + k]);
        i15_cpre[i0 + c + k + 1] = sum + comp;
      }
    }
    __syncthreads();
    // per position: the screened value in both lanes and the tie-run end
    for (int i = tid; i < NL; i += kBThreads) {
      int c = 0;
      while (i >= c_btab.start[c + 1]) ++c;
      if (c_btab.screened[c]) {
        const int i0 = c_btab.start[c], len = c_btab.size[c];
        const unsigned k = i15_map((float)tab[i], i15_s[c], i15_o[c]);
        i15_xq[i] = k | (k << 16);
        const double tol = ldexp(fabs(tab[i]), -44);
        int e = i - i0 + 1;
        while (e < len && fabs(tab[i0 + e] - tab[i]) <= tol) ++e;
        i15_te[i] = (unsigned char)e;
      }
    }
    __syncthreads();
    i15_fill<kBL, 0>(SmemTabs{i15_s, i15_o, tab, i15_cpre, i15_xq, i15_te}, i15_et, false);
  } else if (TAB) {
    for (int i = tid; i < NG * kGraySlots; i += kBThreads)
      sgray[i] = gray_table_entry(&gpre[(i / kGraySlots) * kGroupSlots], (unsigned)(i % kGraySlots), true);
  }
  __syncthreads();

  const double NK = (double)N * o.K;
  const double INF = __longlong_as_double(0x7ff0000000000000ll);
  double ts = 0.0, tc = 0.0;
  const unsigned long long n_pre = 1ull << Dp;
  const unsigned long long per = n_pre >> parts_log2;
  const unsigned long long p0 = (unsigned long long)part * per;
  const int zero = (N >> 10) & tid;  // 0, opaque to the compiler
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
    for (int j0 = 0; j0 < NMID; j0 += NP) {
      double Sn[NP], Xn[NP], base[NP], th[NP];
      int hn[NP];
#pragma unroll
      for (int p = 0; p < NP; ++p) {
        const int j = j0 + p;
        Sn[p] = S * mid_e[j];
        const double Sg = fma(S, mid_c[j], Sig);
        Xn[p] = FL ? fmax(X, S * mid_x[j]) : FLP ? fmin(X, S * mid_x[j]) : 0.0;
        hn[p] = h + mid_h[j];
        base[p] = Sg - NK;
        const double rS = 1.0 / Sn[p];
        th[p] = (AC || AP) ? -base[p] * rS : FL ? Xn[p] * rS : FLP ? fmin(Xn[p], o.K) * rS : 0.0;
      }
      if (TAB) {
        // node value, affine in sA = sum_c w[h+c] A_c and sN = sum_c w[h+c] n_c
        // (the K1 fold forms, bp_exact_fast.cuh)
        double sA[NP], sN[NP];
        if constexpr (I15)
          leaf_block_fold_i15<kBL, 0, DESC>(SmemTabs{i15_s, i15_o, tab, i15_cpre, i15_xq, i15_te},
                                            reinterpret_cast<const uint4*>(i15_xq) + (j0 & zero),
                                            I15Ctx{reinterpret_cast<const char*>(i15_et), i15_xq, i15_te,
                                                   1u | (unsigned)zero, {0.f, 0.f}},
                                            reinterpret_cast<const double2*>(tab) + (j0 & zero),
                                            reinterpret_cast<const char*>(sgray), w, hn, th, sA, sN);
        else
          leaf_block_fold<kBL, NP, 0, DESC>(reinterpret_cast<const double2*>(tab) + (j0 & zero),
                                            reinterpret_cast<const char*>(sgray), w, hn, th, sA, sN);
#pragma unroll
        for (int p = 0; p < NP; ++p) {
          double val;
          if (AC) val = fma(Sn[p], sA[p], base[p] * sN[p]);
          if (AP) val = -fma(Sn[p], sA[p], base[p] * sN[p]);
          if (FL) val = fma(Sn[p], sA[p] - sW2[hn[p]], Xn[p] * (sW1[hn[p]] - sN[p]));
          if (FLP) val = fma(fmax(o.K - Xn[p], 0.0), sW1[hn[p]] - sN[p], fma(o.K, sN[p], -Sn[p] * sA[p]));
          comp_add(ts, tc, val);
        }
      } else {
#pragma unroll
        for (int p = 0; p < NP; ++p) {
          double val = 0.0;
#pragma unroll
          for (int c = 0; c < NC; ++c) {
            const double bc = b_cls[c];
            const double contrib = EC ? bc * fmax(fma(Sn[p], e_cls[c], -o.K), 0.0)
                                      : bc * fmax(fma(-Sn[p], e_cls[c], o.K), 0.0);
            val = fma(w[hn[p] + c], contrib, val);
          }
          comp_add(ts, tc, val);
        }
      }
    }
  }
  // fixed-order CTA reduce: warp shuffle trees, then warp 0 over the 8 warp sums
  warp_comp_reduce(ts, tc);
  if ((tid & 31) == 0) {
    red_s[tid >> 5] = ts;
    red_c[tid >> 5] = tc;
  }
  __syncthreads();
  if (tid < 32) {
    double a = tid < kBThreads / 32 ? red_s[tid] : 0.0, c = tid < kBThreads / 32 ? red_c[tid] : 0.0;
    warp_comp_reduce(a, c);
    if (tid == 0) {
      const double f = (AC || AP) ? 1.0 / N : 1.0;
      partial[blockIdx.x] = make_double2(a * f, c * f);
    }
  }
}

__global__ void k_batch_combine(const double2* __restrict__ partial, BatchLayout lay, double* __restrict__ values) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= lay.n_opts) return;
  const bool in_head = i < lay.n_whole;
  const int parts_log2 = in_head ? lay.base_log2 : lay.tail_log2;
  const long long first = in_head ? ((long long)i << lay.base_log2)
                                  : ((long long)lay.n_whole << lay.base_log2) +
                                        ((long long)(i - lay.n_whole) << lay.tail_log2);
  double s = 0.0, c = 0.0;
  for (int k = 0; k < (1 << parts_log2); ++k) {  // the option's parts in ascending order
    const double2 p = partial[first + k];
    comp_merge(s, c, p.x, p.y);
  }
  values[i] = s + c;
}

BatchLayout batch_layout(int n_opts, int N) {
  static const int forced = [] {
    const char* e = std::getenv("BINPATHS_BATCH_CPO_LOG2");  // diagnostics: uniform CTAs per option
    return e ? std::atoi(e) : -1;
  }();
  const int max_log2 = std::min(4, N - kBL - kBM);  // >= 1 thread prefix per CTA
  int dev = 0, sms = 148, occ = 3;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const long long slots = (long long)sms * occ;  // resident CTAs (k_exact_batch: 3 per SM)
  BatchLayout lay{n_opts, n_opts, 0, 0};
  if (forced >= 0) {
    lay.base_log2 = lay.tail_log2 = std::min(forced, max_log2);
    return lay;
  }
  // few options: enough CTAs to fill the GPU, at most 16 per option
  while (lay.base_log2 < max_log2 && ((long long)n_opts << lay.base_log2) < slots) ++lay.base_log2;
  lay.tail_log2 = lay.base_log2;
  if (lay.base_log2 == 0 && n_opts > slots) {
    // whole waves of one CTA per option, then the remainder split so that its
    // parts fill (at most) one wave of shorter CTAs
    const int rem = (int)(n_opts % slots);
    int t = 0;
    while (t < max_log2 && ((long long)rem << (t + 1)) <= slots) ++t;
    if (rem && t > 0) {
      lay.n_whole = n_opts - rem;
      lay.tail_log2 = t;
    }
  }
  return lay;
}

cudaError_t launch_exact_batch(const BatchOption* opts_dev, const BatchLayout& lay, int N, unsigned kind,
                               double* values_dev, double2* scratch_dev, cudaStream_t st) {
  BatchArgs ba{N, kind, lay};
  const int grid = (int)lay.ctas();
#define BP_B_CASE(K) \
  case K: k_exact_batch<K><<<grid, kBThreads, 0, st>>>(opts_dev, ba, scratch_dev); break;
  switch (kind) {
    BP_B_CASE(kEC) BP_B_CASE(kEP) BP_B_CASE(kAP) BP_B_CASE(kFLP) BP_B_CASE(kAC) BP_B_CASE(kFL)
    default: return cudaErrorInvalidValue;
  }
#undef BP_B_CASE
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  k_batch_combine<<<(lay.n_opts + 255) / 256, 256, 0, st>>>(scratch_dev, lay, values_dev);
  return cudaGetLastError();
}

}  // namespace bp

// Monte Carlo kernels: stratified ("partitioned") MC and its k = 0 special
// case (basic MC), and the shared-sample estimator.
//
// Reference: pkg/src/binpaths/mc.py -- _stratum_stats (:197-213), sampler
// sample_bits (:98-100) keyed by mc_stream(seed, stratum, rep) (:92-95),
// estimate_shared's draw loop (:287-331).
//
// Stream layout (replaces numpy Philox(SeedSequence(seed, spawn_key=(m, rep)))):
//   key     = (seed mod 2^32, seed >> 32)
//   counter = (word block j, draw index i, stream id m, repetition)
//   suffix step w (0-based after the r prefix steps) is bit w % 32 of group
//   g = w / 32.  Level l < 8 of group g is word (8 g + l) % 4 of block
//   (8 g + l) / 4; the step's level-l bit is bit w % 32 of that word.  The
//   first level whose bit is 1 decides the step: up iff bit (31 - l) of
//   thr_t = floor(p_t 2^32) is 1 (level l is first with probability
//   2^-(l+1), so P(up) so far is the top 8 bits of thr_t).  A step with no 1
//   in 8 levels (probability 2^-8) takes its group's next tie word x and goes
//   up iff x < (thr_t << 8) mod 2^32.  P(up) = thr_t / 2^32 exactly; p_t == 1:
//   always.  Tie words: draws 2 j and 2 j + 1 share the pair block with
//   counter (4, j, m, rep); the first tie of group g of draw i (ascending step
//   order) takes its word 2 (i mod 2) + g.  Later ties of the group (the
//   k-th, k >= 1) take word q = 2 (k - 1) + g of the draw's own overflow
//   stream: word q % 4 of block (5 + q / 4, i, m, rep).
// Streams are disjoint by construction and independent of the thread
// mapping, so results do not depend on the grid, the GPU count or timing.
//
// Work items: (rep, stratum, chunk of kChunk draws).  A CTA evaluates one
// item: thread t takes the pairs of draws chunk_base + 2 t + 512 k (+ 1) in
// lock step, keeps shifted sums (n, mean, M2), the CTA merges them with
// Chan's formula in a fixed tree, and a second kernel merges the items of a
// stratum in ascending order.
#include "bp_kernels.h"

namespace bp {

constexpr int kMcThreads = 256;
constexpr unsigned long long kChunk = 4096;  // draws per work item

struct Welford {
  double n, mean, m2;
};

__device__ __forceinline__ Welford chan(const Welford& a, const Welford& b) {
  if (b.n == 0.0) return a;
  if (a.n == 0.0) return b;
  const double n = a.n + b.n;
  const double delta = b.mean - a.mean;
  const double f = b.n / n;
  Welford r;
  r.n = n;
  r.mean = fma(delta, f, a.mean);
  r.m2 = a.m2 + b.m2 + delta * delta * a.n * f;
  return r;
}

// fixed-order CTA merge of per-thread Welford states; thread 0 gets the total
__device__ Welford cta_merge(Welford w) {
  __shared__ double sn[kMcThreads], smean[kMcThreads], sm2[kMcThreads];
  sn[threadIdx.x] = w.n;
  smean[threadIdx.x] = w.mean;
  sm2[threadIdx.x] = w.m2;
  __syncthreads();
  for (int stride = kMcThreads / 2; stride > 0; stride >>= 1) {
    if (threadIdx.x < stride) {
      Welford a{sn[threadIdx.x], smean[threadIdx.x], sm2[threadIdx.x]};
      Welford b{sn[threadIdx.x + stride], smean[threadIdx.x + stride], sm2[threadIdx.x + stride]};
      Welford c = chan(a, b);
      sn[threadIdx.x] = c.n;
      smean[threadIdx.x] = c.mean;
      sm2[threadIdx.x] = c.m2;
    }
    __syncthreads();
  }
  Welford r{sn[0], smean[0], sm2[0]};
  __syncthreads();
  return r;
}

// Path state after the r prefix steps of stratum m (the prefix is fixed).
struct PathState {
  double S, sum, mx, mn;
};

__device__ __forceinline__ double payoff_of(unsigned kind, const PathState& st, double K, double invN) {
  const double mean = st.sum * invN;
  switch (kind) {
    case kEC: return fmax(st.S - K, 0.0);
    case kEP: return fmax(K - st.S, 0.0);
    case kAP: return fmax(K - mean, 0.0);
    case kFLP: return fmax(K - st.mn, 0.0);
    case kAC: return fmax(mean - K, 0.0);
    default: return st.mx - st.S;
  }
}

// Step tables in shared memory.  Byte table: 8 consecutive steps with
// up-pattern b (first step = bit 0): relative price after the 8 steps (e),
// sum of the 8 relative prices (c) in ec[b]; their max (x) and min (n) in
// xn[b].  The nibble table holds the same for 4 steps (the leftover nibble of
// a suffix that is not a multiple of 8 steps).  Built once per CTA.
struct Nib {
  double e, c, x, n;
};
struct McTables {
  double2 ec[256];
  double2 xn[256];
  Nib nib[16];
};

// shared-window address of p, opaque to the compiler so it stays in one
// register instead of being rebuilt (S2UR + ULEA) before every table load
__device__ __forceinline__ uint32_t shared_address(const void* p) {
  uint32_t s = (uint32_t)__cvta_generic_to_shared(p);
  asm volatile("" : "+r"(s));
  return s;
}

__device__ __forceinline__ void build_tables(const McArgs& a, McTables& t) {
  for (int b = threadIdx.x; b < 256; b += blockDim.x) {
    double r = 1.0, c = 0.0, x = -INFINITY, n = INFINITY;
    for (int l = 0; l < 8; ++l) {
      r *= ((b >> l) & 1) ? a.u : a.d;
      c += r;
      x = fmax(x, r);
      n = fmin(n, r);
      if (l == 3 && b < 16) t.nib[b] = Nib{r, c, x, n};
    }
    t.ec[b] = make_double2(r, c);
    t.xn[b] = make_double2(x, n);
  }
}

// State after the r prefix steps of stratum m (bit r - 1 of m is the first
// step), through the step tables: whole bytes, a nibble, then single steps.
__device__ __forceinline__ PathState prefix_state(const McArgs& a, const McTables& tab, unsigned long long m) {
  PathState st{a.S0, 0.0, -INFINITY, INFINITY};
  if (a.r == 0) return st;
  const unsigned long long rev = __brevll(m) >> (64 - a.r);  // first step = bit 0, the tables' order
  auto advance = [&](double e, double c, double x, double n) {
    st.sum = fma(st.S, c, st.sum);
    st.mx = fmax(st.mx, st.S * x);
    st.mn = fmin(st.mn, st.S * n);
    st.S *= e;
  };
  int t = 0;
  for (; t + 8 <= a.r; t += 8) {
    const int b = (int)((rev >> t) & 255ull);
    advance(tab.ec[b].x, tab.ec[b].y, tab.xn[b].x, tab.xn[b].y);
  }
  if (t + 4 <= a.r) {
    const Nib q = tab.nib[(rev >> t) & 15ull];
    advance(q.e, q.c, q.x, q.n);
    t += 4;
  }
  for (; t < a.r; ++t) {
    st.S *= ((rev >> t) & 1ull) ? a.u : a.d;
    st.sum += st.S;
    st.mx = fmax(st.mx, st.S);
    st.mn = fmin(st.mn, st.S);
  }
  return st;
}

constexpr uint32_t kMcPlaneBlocks = kMcLevels / 4;     // Philox blocks per group of 32 steps
constexpr uint32_t kMcTieBlock0 = 2 * kMcPlaneBlocks;  // first block of the tie words

// The up/down bits of the suffix steps of NS draws (i0, i0 + stride, ...) on
// stream (m, rep): B[d][g] bit b = step 32 g + b of draw d goes up.
//
// Each step is Bernoulli(thr_t / 2^32), exactly: level l's word gives every
// one of the 32 steps of a group a fair bit, the first level whose bit is 1
// decides the step (up iff the threshold's bit 31 - l is 1), the others stay
// open.  The open sets U_0 > U_1 > ... are nested, so the up set is
// XOR_l (U_l & C_l) with C_l = T_l ^ T_{l+1} the planes where the threshold
// bit flips (T_0 = T_9 = 0): 2 LOP3 per level and group instead of a compare
// per step.  After kMcLevels levels an open step (probability 2^-kMcLevels)
// takes the group's next tie word x and goes up iff
// x < (thr_t << kMcLevels) mod 2^32.  5 Philox blocks per draw instead of
// one word per step (13 blocks at 52 steps).
//
// Tie words: draws 2 j and 2 j + 1 share one pair block (4 words: 2 draws x
// 2 groups) for the first tie of each group, so a thread walking the two
// draws of a pair in lock step computes 4 + 1/2 Philox blocks per draw.
// CONSTP (every suffix step has the same threshold): the first tie of a
// group needs no bit search -- the lowest open bit u & -u goes up iff its
// word is below the common tie threshold.  Second and later ties of a group
// (about 1 draw in 150) take words of the draw's own overflow blocks.
template <bool CONSTP, int G>
__device__ __forceinline__ void resolve_ties(const McArgs& a, uint32_t& Bg, uint32_t u, uint32_t x0, uint32_t thr_tie,
                                             uint32_t draw, uint32_t stream, uint32_t rep) {
  auto tie_thr = [&](uint32_t low) -> uint32_t {
    if (CONSTP) return thr_tie;
    return a.thr[a.r + 32 * G + (__ffs((int)low) - 1)] << kMcLevels;
  };
  const uint32_t first = u & (0u - u);
  if (CONSTP) {
    if (x0 < thr_tie) Bg |= first;
  } else if (u) {
    if (x0 < tie_thr(first)) Bg |= first;
  }
  if (u == first) return;
  u ^= first;
  uint32_t blk[4] = {0u, 0u, 0u, 0u};
  for (uint32_t k = 1; u; ++k, u &= u - 1u) {
    const uint32_t q = 2u * (k - 1u) + G;
    if ((q & 3u) == (uint32_t)G) philox4x32_10_rk(kMcTieBlock0 + 1u + (q >> 2), draw, stream, rep, a.rk, blk);
    const uint32_t x = (q & 2u) ? blk[2 + G] : blk[G];
    const uint32_t low = u & (0u - u);
    if (x < tie_thr(low)) Bg |= low;
  }
}

// NS == 1: any draw i0.  NS even: the consecutive draws i0 .. i0 + NS - 1, i0 even.
template <bool CONSTP, int NS>
__device__ __forceinline__ void draw_bits(const McArgs& a, uint32_t (&B)[NS][2], uint32_t i0, uint32_t stream,
                                          uint32_t rep) {
  static_assert(NS == 1 || NS % 2 == 0, "draws are walked singly or in whole pairs");
  const int nsuf = a.N - a.r;
  uint32_t U[NS][2];
#pragma unroll
  for (int g = 0; g < 2; ++g) {
#pragma unroll
    for (int d = 0; d < NS; ++d) {
      B[d][g] = a.bits0[g];
      U[d][g] = a.open[g];
    }
    if (32 * g < nsuf) {
#pragma unroll
      for (int jb = 0; jb < (int)kMcPlaneBlocks; ++jb) {
        uint32_t blk[NS][4];
#pragma unroll
        for (int d = 0; d < NS; ++d) philox4x32_10_rk(g * kMcPlaneBlocks + jb, i0 + d, stream, rep, a.rk, blk[d]);
#pragma unroll
        for (int l = 0; l < 4; ++l) {
          const uint32_t C = a.flip[g][4 * jb + l];
#pragma unroll
          for (int d = 0; d < NS; ++d) {
            U[d][g] &= ~blk[d][l];
            B[d][g] ^= U[d][g] & C;
          }
        }
      }
    }
  }
  const uint32_t thr_tie = a.thr[a.r < a.N ? a.r : 0] << kMcLevels;
  constexpr int NP = NS == 1 ? 1 : NS / 2;
  uint32_t tie[NP][4];
#pragma unroll
  for (int pr = 0; pr < NP; ++pr) philox4x32_10_rk(kMcTieBlock0, (i0 >> 1) + pr, stream, rep, a.rk, tie[pr]);
#pragma unroll
  for (int d = 0; d < NS; ++d) {
    uint32_t x0, x1;
    if (NS == 1) {
      x0 = (i0 & 1u) ? tie[0][2] : tie[0][0];
      x1 = (i0 & 1u) ? tie[0][3] : tie[0][1];
    } else {
      x0 = tie[d / 2][2 * (d & 1)];
      x1 = tie[d / 2][2 * (d & 1) + 1];
    }
    resolve_ties<CONSTP, 0>(a, B[d][0], U[d][0], x0, thr_tie, i0 + d, stream, rep);
    resolve_ties<CONSTP, 1>(a, B[d][1], U[d][1], x1, thr_tie, i0 + d, stream, rep);
  }
}

// Walk the N - r suffix steps of NS draws (draw_bits: one draw, or whole
// pairs) in lock step from their states (the Philox rounds of the NS
// counters interleave, giving the scheduler independent work).  Full blocks of 4 steps use the nibble tables; the
// tail walks step by step.
template <unsigned KIND, bool CONSTP, int NS>
__device__ __forceinline__ void walk_suffix_n(const McArgs& a, const McTables& tab, uint32_t tab_s, PathState (&s)[NS],
                                              uint32_t i0, uint32_t stream, uint32_t rep) {
  constexpr bool need_max = KIND == kFL;
  constexpr bool need_min = KIND == kFLP;
  constexpr bool need_sum = KIND == kAC || KIND == kAP;
  const int nsuf = a.N - a.r;
  const int nbytes = nsuf >> 3;
  uint32_t B[NS][2];
  draw_bits<CONSTP, NS>(a, B, i0, stream, rep);
  auto advance = [&](PathState& st, double e, double c, double x, double n) {
    if (need_sum) st.sum = fma(st.S, c, st.sum);
    if (need_max) st.mx = fmax(st.mx, st.S * x);
    if (need_min) st.mn = fmin(st.mn, st.S * n);
    st.S *= e;
  };
  // whole bytes of 8 steps, one table entry each: entry address = table
  // base + 16 x byte (PRMT + LEA; tab_s is the table's shared-window address,
  // made once per kernel)
  auto byte_step = [&](int g, int k) {
#pragma unroll
    for (int d = 0; d < NS; ++d) {
      const uint32_t addr = tab_s + (__byte_perm(B[d][g], 0u, 0x4440u + k) << 4);
      double e, c, x = 0.0, n = 0.0;
      asm("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(e), "=d"(c) : "r"(addr));
      if (need_max || need_min) asm("ld.shared.v2.f64 {%0, %1}, [%2+4096];" : "=d"(x), "=d"(n) : "r"(addr));
      advance(s[d], e, c, x, n);
    }
  };
#pragma unroll
  for (int g = 0; g < 2; ++g) {
    const int cnt = nbytes - 4 * g;
    if (cnt >= 4) {  // a whole group: no per-byte test
#pragma unroll
      for (int k = 0; k < 4; ++k) byte_step(g, k);
    } else {
#pragma unroll
      for (int k = 0; k < 3; ++k)
        if (k < cnt) byte_step(g, k);
    }
  }
  // a leftover nibble, then up to 3 single steps
  int w = 8 * nbytes;
  if (nsuf - w >= 4) {
#pragma unroll
    for (int d = 0; d < NS; ++d) {
      const Nib q = tab.nib[(((w >> 5) ? B[d][1] : B[d][0]) >> (w & 31)) & 15u];
      advance(s[d], q.e, q.c, q.x, q.n);
    }
    w += 4;
  }
  for (; w < nsuf; ++w) {
#pragma unroll
    for (int d = 0; d < NS; ++d) {
      const uint32_t word = (w >> 5) ? B[d][1] : B[d][0];
      s[d].S *= ((word >> (w & 31)) & 1u) ? a.u : a.d;
      if (need_sum) s[d].sum += s[d].S;
      if (need_max) s[d].mx = fmax(s[d].mx, s[d].S);
      if (need_min) s[d].mn = fmin(s[d].mn, s[d].S);
    }
  }
}

template <unsigned KIND, bool CONSTP>
__device__ __forceinline__ PathState walk_suffix(const McArgs& a, const McTables& tab, uint32_t tab_s, PathState st, uint32_t i,
                                                 uint32_t stream, uint32_t rep) {
  PathState s[1] = {st};
  walk_suffix_n<KIND, CONSTP, 1>(a, tab, tab_s, s, i, stream, rep);
  return s[0];
}

#ifndef BP_MC_NS
#define BP_MC_NS 2  // draws per thread in lock step (K4; even: whole pairs; r2 scan: 2 and 4 within 1 %)
#endif
constexpr int kMcNS = BP_MC_NS;

// Per-thread running statistics without a per-draw division: sums of
// (v - c) and (v - c)^2 around the thread's first value c (no cancellation
// problem: c is an actual sample), turned into (n, mean, M2) once.
struct ShiftedSums {
  double c, s1, s2, n;
  __device__ __forceinline__ void add(double v) {
    if (n == 0.0) c = v;
    const double d = v - c;
    s1 += d;
    s2 = fma(d, d, s2);
    n += 1.0;
  }
  __device__ __forceinline__ Welford welford() const {
    if (n == 0.0) return Welford{0.0, 0.0, 0.0};
    const double m1 = s1 / n;
    return Welford{n, c + m1, fmax(s2 - s1 * m1, 0.0)};
  }
};

// ---------------------------------------------------------------------------
// K4/K5: one CTA per work item (grid-stride).  item -> (rep k, stratum m, first draw)
#ifndef BP_MC_MINB
#define BP_MC_MINB 4  // resident CTAs per SM targeted by K4 (r2 scan with the bit-sliced sampler: 1-3 lose 7-20 %)
#endif
template <unsigned KIND, bool CONSTP>
__global__ void __launch_bounds__(kMcThreads, BP_MC_MINB)
k_mc_strata(const __grid_constant__ McArgs a, const unsigned long long* __restrict__ draws,
            const unsigned long long* __restrict__ item_stratum, const unsigned long long* __restrict__ item_first,
            unsigned long long items_per_rep, int n_reps, double* __restrict__ item_out) {
  __shared__ __align__(16) McTables tab;
  build_tables(a, tab);
  const uint32_t tab_s = shared_address(&tab);
  __syncthreads();
  const unsigned long long n_items = items_per_rep * (unsigned long long)n_reps;
  for (unsigned long long it = blockIdx.x; it < n_items; it += gridDim.x) {
    const unsigned long long k = it / items_per_rep, li = it % items_per_rep;
    const unsigned long long m = item_stratum[li];
    const unsigned long long first = item_first[li];
    const unsigned long long R = draws[m];
    const unsigned long long last = first + kChunk < R ? first + kChunk : R;
    const PathState pre = prefix_state(a, tab, m);
    ShiftedSums acc{0.0, 0.0, 0.0, 0.0};
    // whole pairs (2 j, 2 j + 1) in groups of kMcNS consecutive draws per
    // thread, then the remaining draws one per thread; an item starting at an
    // odd draw (bp_mc_range with an unaligned range) walks them all singly
    unsigned long long single0 = first;
    if ((first & 1ull) == 0ull) {
      const unsigned long long span = (unsigned long long)kMcNS * kMcThreads;
      const unsigned long long whole = (last - first) / span * span;
      for (unsigned long long i = first + (unsigned long long)kMcNS * threadIdx.x; i < first + whole; i += span) {
        PathState sd[kMcNS];
#pragma unroll
        for (int d = 0; d < kMcNS; ++d) sd[d] = pre;
        walk_suffix_n<KIND, CONSTP, kMcNS>(a, tab, tab_s, sd, (uint32_t)i, (uint32_t)m, a.rep0 + (uint32_t)k);
#pragma unroll
        for (int d = 0; d < kMcNS; ++d) acc.add(payoff_of(KIND, sd[d], a.K, a.invN));
      }
      single0 = first + whole;
    }
    for (unsigned long long i = single0 + threadIdx.x; i < last; i += kMcThreads) {
      const PathState st = walk_suffix<KIND, CONSTP>(a, tab, tab_s, pre, (uint32_t)i, (uint32_t)m, a.rep0 + (uint32_t)k);
      acc.add(payoff_of(KIND, st, a.K, a.invN));
    }
    const Welford t = cta_merge(acc.welford());
    if (threadIdx.x == 0) {
      item_out[it * 3 + 0] = t.n;
      item_out[it * 3 + 1] = t.mean;
      item_out[it * 3 + 2] = t.m2;
    }
  }
}

// ascending-order merge of a stratum's items -> theta, sse
__global__ void k_mc_strata_merge(const double* __restrict__ item_out, const unsigned long long* __restrict__ stratum_item0,
                                  unsigned long long items_per_rep, int n_strata, int n_reps,
                                  double* __restrict__ theta, double* __restrict__ sse) {
  const long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (idx >= (long long)n_strata * n_reps) return;
  const long long k = idx / n_strata, m = idx % n_strata;
  const unsigned long long i0 = stratum_item0[m], i1 = stratum_item0[m + 1];
  Welford acc{0.0, 0.0, 0.0};
  for (unsigned long long i = i0; i < i1; ++i) {
    const unsigned long long it = (unsigned long long)k * items_per_rep + i;
    Welford b{item_out[it * 3], item_out[it * 3 + 1], item_out[it * 3 + 2]};
    acc = chan(acc, b);
  }
  theta[idx] = acc.n > 0.0 ? acc.mean : 0.0;
  sse[idx] = acc.n > 0.0 ? acc.m2 : 0.0;
}

// item -> (stratum, first draw) lists, one thread per stratum
__global__ void k_mc_items(const unsigned long long* __restrict__ draws, const unsigned long long* __restrict__ first,
                           const unsigned long long* __restrict__ stratum_item0, int n_strata,
                           unsigned long long* __restrict__ item_stratum, unsigned long long* __restrict__ item_first) {
  const int m = blockIdx.x * blockDim.x + threadIdx.x;
  if (m >= n_strata) return;
  unsigned long long it = stratum_item0[m];
  for (unsigned long long f = first ? first[m] : 0ull; f < draws[m]; f += kChunk, ++it) {
    item_stratum[it] = (unsigned long long)m;
    item_first[it] = f;
  }
}

cudaError_t launch_mc_items(const unsigned long long* draws_dev, const unsigned long long* first_dev,
                            const unsigned long long* stratum_item0_dev, int n_strata,
                            unsigned long long* item_stratum_dev, unsigned long long* item_first_dev,
                            cudaStream_t st) {
  k_mc_items<<<(n_strata + 127) / 128, 128, 0, st>>>(draws_dev, first_dev, stratum_item0_dev, n_strata,
                                                     item_stratum_dev, item_first_dev);
  return cudaGetLastError();
}

cudaError_t launch_mc_strata(const McArgs& a, const unsigned long long* draws_dev,
                             const unsigned long long* item_stratum_dev, const unsigned long long* item_first_dev,
                             unsigned long long items_per_rep, int n_reps, int n_strata, double* item_out_dev,
                             double* theta_dev, double* sse_dev, const unsigned long long* stratum_item0_dev,
                             cudaStream_t st) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const unsigned long long n_items = items_per_rep * (unsigned long long)n_reps;
  // one threshold for every stream-decided suffix step (the BASELINE trees)
  bool constp = a.r < a.N && !((a.always[a.r / 32] >> (a.r % 32)) & 1u);
  for (int t = a.r; t < a.N && constp; ++t)
    if (!((a.always[t / 32] >> (t % 32)) & 1u)) constp = a.thr[t] == a.thr[a.r];
  if (n_items) {
    const int grid = (int)(n_items < (unsigned long long)sms * 16 ? n_items : (unsigned long long)sms * 16);
#define BP_MC_CASE(K)                                                                                         \
  case K:                                                                                                     \
    if (constp)                                                                                               \
      k_mc_strata<K, true><<<grid, kMcThreads, 0, st>>>(a, draws_dev, item_stratum_dev, item_first_dev,       \
                                                         items_per_rep, n_reps, item_out_dev);                 \
    else                                                                                                      \
      k_mc_strata<K, false><<<grid, kMcThreads, 0, st>>>(a, draws_dev, item_stratum_dev, item_first_dev,      \
                                                          items_per_rep, n_reps, item_out_dev);                \
    break;
    switch (a.kind) {
      BP_MC_CASE(kEC) BP_MC_CASE(kEP) BP_MC_CASE(kAP) BP_MC_CASE(kFLP) BP_MC_CASE(kAC) BP_MC_CASE(kFL)
      default: return cudaErrorInvalidValue;
    }
#undef BP_MC_CASE
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  const long long total = (long long)n_strata * n_reps;
  k_mc_strata_merge<<<(unsigned)((total + 255) / 256), 256, 0, st>>>(item_out_dev, stratum_item0_dev, items_per_rep,
                                                                      n_strata, n_reps, theta_dev, sse_dev);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Shared-sample MC: draw i's suffix is drawn once (stream 0) and evaluated
// under all M prefixes.  Per item: Welford of the inner sums + per-warp,
// per-stratum payoff sums (fixed order, no atomics).
template <unsigned KIND>
__global__ void __launch_bounds__(kMcThreads)
k_mc_shared(const __grid_constant__ McArgs a, unsigned long long R, const double* __restrict__ masses,
            const double* __restrict__ pre_tab /* [M][4] S, sum, mx, mn after r steps */, int M,
            unsigned long long items_per_rep, int n_reps, double* __restrict__ item_out,
            double* __restrict__ warp_sums /* [item][8][M] */) {
  __shared__ __align__(16) McTables tab;
  build_tables(a, tab);
  const uint32_t tab_s = shared_address(&tab);
  __syncthreads();
  const unsigned long long n_items = items_per_rep * (unsigned long long)n_reps;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (unsigned long long it = blockIdx.x; it < n_items; it += gridDim.x) {
    const unsigned long long k = it / items_per_rep, li = it % items_per_rep;
    const unsigned long long first = li * kChunk;
    const unsigned long long last = first + kChunk < R ? first + kChunk : R;
    double* ws = warp_sums + (it * 8 + warp) * (unsigned long long)M;
    for (int m = lane; m < M; m += 32) ws[m] = 0.0;
    __syncwarp();
    Welford w{0.0, 0.0, 0.0};
    // iterate in warp-synchronous rounds so the per-stratum warp reduce is uniform
    for (unsigned long long base = first + warp * 32; base < last; base += kMcThreads) {
      const unsigned long long i = base + lane;
      const bool live = i < last;
      // suffix relative to a unit start price
      PathState rel{1.0, 0.0, -INFINITY, INFINITY};
      if (live) rel = walk_suffix<KIND, false>(a, tab, tab_s, rel, (uint32_t)i, 0u, a.rep0 + (uint32_t)k);
      double inner = 0.0;
      for (int m = 0; m < M; ++m) {
        const double S = pre_tab[4 * m], sum = pre_tab[4 * m + 1], mx = pre_tab[4 * m + 2], mn = pre_tab[4 * m + 3];
        PathState st{S * rel.S, fma(S, rel.sum, sum), fmax(mx, S * rel.mx), fmin(mn, S * rel.mn)};
        const double v = live ? payoff_of(KIND, st, a.K, a.invN) : 0.0;
        inner = fma(masses[m], v, inner);
        double s = v;
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
        if (lane == 0) ws[m] += s;
      }
      if (live) {
        w.n += 1.0;
        const double delta = inner - w.mean;
        w.mean += delta / w.n;
        w.m2 = fma(delta, inner - w.mean, w.m2);
      }
    }
    const Welford t = cta_merge(w);
    if (threadIdx.x == 0) {
      item_out[it * 3 + 0] = t.n;
      item_out[it * 3 + 1] = t.mean;
      item_out[it * 3 + 2] = t.m2;
    }
    __syncthreads();
  }
}

__global__ void k_mc_shared_merge(const double* __restrict__ item_out, const double* __restrict__ warp_sums,
                                  unsigned long long items_per_rep, int M, int n_reps, double Rd,
                                  double* __restrict__ inner_mean, double* __restrict__ inner_sse,
                                  double* __restrict__ stratum_means) {
  const long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (idx < n_reps) {
    Welford acc{0.0, 0.0, 0.0};
    for (unsigned long long i = 0; i < items_per_rep; ++i) {
      const unsigned long long it = (unsigned long long)idx * items_per_rep + i;
      acc = chan(acc, Welford{item_out[it * 3], item_out[it * 3 + 1], item_out[it * 3 + 2]});
    }
    inner_mean[idx] = acc.mean;
    inner_sse[idx] = acc.m2;
  }
  if (idx < (long long)M * n_reps) {
    const long long k = idx / M, m = idx % M;
    double s = 0.0, c = 0.0;
    for (unsigned long long i = 0; i < items_per_rep; ++i)
      for (int wp = 0; wp < 8; ++wp)
        comp_add(s, c, warp_sums[(((unsigned long long)k * items_per_rep + i) * 8 + wp) * (unsigned long long)M + m]);
    stratum_means[idx] = (s + c) / Rd;
  }
}

cudaError_t launch_mc_shared(const McArgs& a, unsigned long long R, const double* masses_dev, const double* pre_tab_dev,
                             int M, int n_reps, double* item_out_dev, double* warp_sums_dev,
                             unsigned long long items_per_rep, double* inner_mean_dev, double* inner_sse_dev,
                             double* stratum_means_dev, cudaStream_t st) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const unsigned long long n_items = items_per_rep * (unsigned long long)n_reps;
  const int grid = (int)(n_items < (unsigned long long)sms * 16 ? n_items : (unsigned long long)sms * 16);
#define BP_SH_CASE(K) \
  case K: k_mc_shared<K><<<grid, kMcThreads, 0, st>>>(a, R, masses_dev, pre_tab_dev, M, items_per_rep, n_reps, item_out_dev, warp_sums_dev); break;
  switch (a.kind) {
    BP_SH_CASE(kEC) BP_SH_CASE(kEP) BP_SH_CASE(kAP) BP_SH_CASE(kFLP) BP_SH_CASE(kAC) BP_SH_CASE(kFL)
    default: return cudaErrorInvalidValue;
  }
#undef BP_SH_CASE
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  const long long total = (long long)M * n_reps > n_reps ? (long long)M * n_reps : n_reps;
  k_mc_shared_merge<<<(unsigned)((total + 255) / 256), 256, 0, st>>>(item_out_dev, warp_sums_dev, items_per_rep, M,
                                                                      n_reps, (double)R, inner_mean_dev, inner_sse_dev,
                                                                      stratum_means_dev);
  return cudaGetLastError();
}

unsigned long long mc_chunk() { return kChunk; }

}  // namespace bp

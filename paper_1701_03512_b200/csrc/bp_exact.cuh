// Exact 2^N path enumeration on B200 (sm_100a).
//
// Replaces the reference hot loop _rank_value (pkg/src/binpaths/exact.py:83-100),
// which materialises a bool[CHUNK, N] bit matrix (paths.py:170-173), a row
// product of per-step probabilities (exact.py:95) and a cumprod of the price
// path (payoffs.py:103-104) for every path.
//
// Index decomposition (path code, step 1 = most significant bit, paths.py:1-12):
//
//   code = [ super-block | unit | lane | middle (m bits) | inner block (L bits) ]
//           \____________ node index (D = N - L bits) ____________/
//
// * a warp owns a UNIT of 32 * 2^m consecutive nodes; lane i owns the 2^m
//   nodes whose top D - m bits are (unit, i) -- its thread prefix;
// * the thread walks its prefix once (S, running sum, max, min, up count),
//   then visits its 2^m nodes with the middle tables (mid_*), then every
//   leaf of each node in a fully unrolled block of 2^L leaves;
// * every leaf is evaluated explicitly with ONE compare; the affine structure
//   of the payoffs makes the compare the whole payoff decision:
//     Asian:    sum_j S_j = Sig_node + S_node * c_s   (c_s = sum of the L
//               relative prices of inner suffix s, a table)
//     lookback: max_j S_j = max(Mx_node, S_node * mx_s)
//   so "payoff > 0" is "c_s > theta_node" with theta = (N K - Sig)/S, and an
//   in-the-money leaf contributes S c_s + (Sig - N K).
// * the inner table is laid out by up-count class c = |s| and, inside a
//   class, sorted in the compare direction (host side, per tree), then cut
//   into groups of <= kGroup positions.  Inside a group the in-the-money leaves
//   are therefore a prefix: the per-leaf compares (DSETP + predicated
//   increment, in independent chains of kChain leaves) give the count n, and
//   the group's contribution sum_ITM c_s is the precomputed prefix sum P_g[n]
//   (one shared-memory load per group).
//   Per class the node keeps A_c = sum of ITM values and n_c = ITM count;
//   the node value is sum_c w[h + c] (S A_c + base n_c), w[h] =
//   e^{-qT} p^h (1-p)^{N-h} (exact.py:95,99 folded into one table).
#pragma once
#include <cmath>
#include <cstdint>
#include <cstring>
#include "bp_common.cuh"

namespace bp {

// kind bit positions (include/binpaths_b200.h: bp_payoff)
enum KindBit : int { kEC = 0, kEP = 1, kAP = 2, kFLP = 3, kAC = 4, kFL = 5 };
constexpr int kNumKinds = 6;

// table slot used by a kind in the fast engine; -1 = no per-leaf table
BP_HD constexpr int kind_table(int k) {
  return (k == kAC || k == kAP) ? 0 : (k == kFL) ? 1 : (k == kFLP) ? 2 : -1;
}

constexpr int kMidMax = 64;          // 2^m, m <= 6
constexpr int kUnitTargetLog2 = 14;  // units >= 2^14 when the tree allows it (r1 scan)
// K1 (units handed out dynamically): units >= 2^13 when the tree allows it
// (r2 scan, N = 30: 2^13 units of 8 nodes per lane beat 2^14 of 4 by 2-4 %)
constexpr int kFastUnitTargetLog2 = 13;
constexpr int kMidCap = 5;           // at most 2^kMidCap middle nodes per lane per unit (BINPATHS_MID_CAP; r2 scan)
constexpr int kMaxSB = 64;           // canonical super-blocks (top 6 bits of the unit index)
constexpr int kFastMinN = 16;        // smaller trees use the per-path walk

struct ExactScalars {
  double S0, K, NK, u, d, invN;
  int N, L, D, m, Dp, n_mid;
  int q;             // a unit is 2^q consecutive 32-lane prefix groups
  int zero;          // opaque 0 (defeats constant hoisting in the leaf loop)
  unsigned long long unit_first, unit_end;
};

// binomial coefficients and the class / group layout of the inner block
// (iterative constexpr: usable in templates, host and device code)
__host__ __device__ constexpr int binom(int n, int k) {
  if (k < 0 || k > n) return 0;
  long long r = 1;
  for (int i = 1; i <= k; ++i) r = r * (n - k + i) / i;
  return (int)r;
}
__host__ __device__ constexpr int class_start(int L, int c) {
  int s = 0;
  for (int i = 0; i < c; ++i) s += binom(L, i);
  return s;
}
// Leaves per sorted group (prefix-sum lookup granularity) and leaves per
// independent count chain inside a group: 32 / 4 measured best for K1 (both
// the one- and two-table kernels) and K3 (profiles/r1_scan_group_chains*.log;
// 8 / 8 before: 7 % slower).
#ifndef BP_GROUP
#define BP_GROUP 32
#endif
constexpr int kGroup = BP_GROUP;
#ifndef BP_CHAIN
#define BP_CHAIN 4
#endif
constexpr int kChain = BP_CHAIN;
__host__ __device__ constexpr int class_groups(int L, int c) { return (binom(L, c) + kGroup - 1) / kGroup; }
__host__ __device__ constexpr int group_base(int L, int c) {
  int s = 0;
  for (int i = 0; i < c; ++i) s += class_groups(L, i);
  return s;
}
__host__ __device__ constexpr int n_groups(int L) { return group_base(L, L + 1); }
constexpr int kGroupSlots = kGroup + 1;  // prefix sums for n = 0..kGroup

// K1 leaf-block configuration (shared by the kernels and the host layout):
// BP_GRAY  -- leaf counts: 0 = predicated increments in chains of kChain,
//             1 = Gray-code predicate chains (bp_gray.cuh);
// BP_FOLD  -- 1 = each class folds into two per-node sums right after its
//             groups (Gray mode only);
// BP_NP    -- nodes per leaf block: every table load feeds NP compares.
#ifndef BP_GRAY
#define BP_GRAY 1
#endif
#ifndef BP_FOLD
#define BP_FOLD 1
#endif
#ifndef BP_NP
#define BP_NP 2
#endif
constexpr int kNodesPerBlock = BP_NP;
constexpr int kNodesPerBlockLog2 = BP_NP == 4 ? 2 : BP_NP == 2 ? 1 : 0;
static_assert(BP_NP == 1 || BP_NP == 2 || BP_NP == 4, "BP_NP must be 1, 2 or 4");

// BP_I15 -- the big classes (>= kI15Min leaves) of the K1 leaf block (L = 8,
//           two nodes per block, fold mode) screen their leaves with a 15-bit
//           fixed-point compare: two nodes per 32-bit integer multiply-add,
//           the sign bits XOR-ed into Gray-code counters, and the rare
//           ambiguous boundary leaf resolved in fp64 (bp_leaf.cuh, I15Class).
#ifndef BP_I15
#define BP_I15 1
#endif
constexpr int kI15Min = 16;
template <int L>
__host__ __device__ constexpr bool i15_on() {
  return BP_I15 && BP_FOLD && BP_GRAY && (L == 8 || L == 9) && kNodesPerBlock == 2;
}
__host__ __device__ constexpr bool i15_class(int L, int c) { return binom(L, c) >= kI15Min; }
__host__ __device__ constexpr int bit_length(int v) {
  int b = 0;
  while (v >> b) ++b;
  return b;
}
// Gray-code counter slots of a class (codes of the counts 0..|c|) and their
// offset in the per-slot entry table
__host__ __device__ constexpr int i15_slots(int L, int c) { return 1 << bit_length(binom(L, c)); }
__host__ __device__ constexpr int i15_base(int L, int c) {
  int s = 0;
  for (int i = 0; i < c; ++i)
    if (i15_class(L, i)) s += i15_slots(L, i);
  return s;
}
__host__ __device__ constexpr int i15_entries(int L) { return i15_base(L, L + 1); }

// The monotone map of the screen: v -> k in [0, 32767], k = clamp(round(vf *
// s + o)) evaluated in fp32 with one fused multiply-add (o carries 1.5 * 2^23,
// so the fp32 result is an integer).  Host (table values) and device (node
// thresholds) evaluate the same IEEE operations, so v1 <= v2 implies
// k(v1) <= k(v2) for s > 0 (>= for s < 0): k(x) > k(theta) proves x > theta,
// k(x) < k(theta) proves x < theta, and only k(x) == k(theta) is ambiguous.
// A NaN threshold maps to 32767 (no leaf is screened in).
constexpr float kI15Magic = 12582912.0f;
__host__ __device__ inline unsigned i15_map(float vf, float s, float o) {
#ifdef __CUDA_ARCH__
  float f = __fmaf_rn(vf, s, o);
  f = fmaxf(fminf(f, kI15Magic + 32767.0f), kI15Magic);
  return __float_as_uint(f) - 0x4B400000u;
#else
  float f = std::fma(vf, s, o);
  f = std::fmax(std::fmin(f, kI15Magic + 32767.0f), kI15Magic);
  unsigned u;
  std::memcpy(&u, &f, sizeof u);
  return u - 0x4B400000u;
#endif
}

// K1's shared-memory tables as one contiguous image (byte offsets), a
// function of (L, kind mask): the host builds the image once per lattice
// (bp_capi.cu build_smem_image) after the argument block, and every CTA
// copies it with coalesced 16-byte loads instead of computing the tables.
__host__ __device__ constexpr size_t align16(size_t v) { return (v + 15) & ~(size_t)15; }
struct K1SmemLayout {
  bool need_w;
  int nt;
  bool i15[2];            // per table slot: the I15 screen on its big classes
  bool lookback[2];       // per table slot: a lookback kind (thresholds tie with the table)
  int ng[2];              // Gray-table groups per slot (I15: only the small classes')
  size_t sw, sW1, sW2;
  size_t sgray[2], si15[2], sxq[2], ste[2], total;
};
__host__ __device__ constexpr int kind_tables(unsigned km) {
  return (int)((km >> kAC) & 1) + (int)((km >> kAP) & 1) + (int)((km >> kFL) & 1) + (int)((km >> kFLP) & 1);
}
#ifndef BP_I15_LOOKBACK
#define BP_I15_LOOKBACK 1  // the screen on the lookback slots too (branch-free boundary fix)
#endif
template <int L>
__host__ __device__ constexpr K1SmemLayout k1_smem_layout(unsigned km) {
  K1SmemLayout o{};
  o.nt = kind_tables(km);
  o.need_w = ((km >> kFL) & 1) || ((km >> kFLP) & 1);
  // table slots in kind order AC, AP, FL, FLP
  int kinds[2] = {-1, -1}, t = 0;
  const int order[4] = {kAC, kAP, kFL, kFLP};
  for (int i = 0; i < 4; ++i)
    if (((km >> order[i]) & 1) && t < 2) kinds[t++] = order[i];
  int small = 0;
  for (int c = 0; c <= L; ++c)
    if (!i15_class(L, c)) small += class_groups(L, c);
  constexpr int kSlots = 64;  // Gray-table slots per group (kGraySlots, bp_leaf.cuh)
  size_t off = 0;
  o.sw = off;
  off = align16(off + sizeof(double) * (kMaxN + 2 + L + 1));
  o.sW1 = off;
  off += o.need_w ? sizeof(double) * (kMaxN + 2) : 0;
  o.sW2 = off;
  off = align16(off + (o.need_w ? sizeof(double) * (kMaxN + 2) : 0));
  for (int s = 0; s < 2; ++s) {
    const bool has = s < o.nt;
    o.lookback[s] = has && (kinds[s] == kFL || kinds[s] == kFLP);
    o.i15[s] = has && i15_on<L>() && (!o.lookback[s] || BP_I15_LOOKBACK);
    o.ng[s] = has ? (o.i15[s] ? small : n_groups(L)) : 0;
    o.sgray[s] = off;
    off += (size_t)16 * o.ng[s] * kSlots;
    o.si15[s] = off;
    off += o.i15[s] ? (size_t)(o.lookback[s] ? 48 : 32) * i15_entries(L) : 0;  // i15_entry_bytes (bp_leaf.cuh)
    o.sxq[s] = off;
    off += o.i15[s] ? (size_t)4 << L : 0;
    o.ste[s] = off;
    off = align16(off + (o.i15[s] ? (size_t)1 << L : 0));
  }
  o.total = align16(off);
  return o;
}

// K1's kernel parameter block: what the leaf loops read with uniform loads.
// The tables only the CTA setup or the rare exact walk need live in the
// device image after it (ExactTables + the shared-memory image).
template <int L>
struct __align__(16) ExactArgs {
  // inner tables by position (class-major, sorted in the compare direction
  // inside a class), slot-major: tab[slot * 2^L + i]
  double tab[2 << L];
  double mid_c[kMidMax], mid_e[kMidMax], mid_mx[kMidMax], mid_mn[kMidMax];
  int mid_h[kMidMax];
  double w[kMaxN + 2];    // e^{-qT} p^h (1-p)^{N-h}, h = 0..N (zero padded)
  double e_cls[L + 1];    // S_N / S_node for an inner suffix with c ups
  double b_cls[L + 1];    // leaves per class, C(L, c)
  // I15 screen: per slot and class, the monotone map (scale, offset)
  float nrm_s[2][L + 1], nrm_o[2][L + 1];
  ExactScalars s;
};

// Host-side tables of a K1 argument block (built with it): the group prefix
// sums of the Gray tables and, for the I15 screen, per slot the screened
// value k of every position in both 16-bit lanes (k | k << 16), the end
// (exclusive, class-relative) of the tie run starting at each position (the
// following positions within 2^-44 relative: a leaf whose value ties with
// the threshold's to that precision contributes the same either way, so a
// tie run is classified as one leaf) and the class prefix sums P_c[n],
// n = 0..|c|, at cpre[slot][class_start(L, c) + c + n].  cpre also travels
// to the device after the shared-memory image (the exact walk reads it).
template <int L>
struct ExactTables {
  double gpre[2][n_groups(L)][kGroupSlots];
  unsigned xq[2][1 << L];
  unsigned char te[2][1 << L];
  double cpre[2][(1 << L) + L + 1];
};
template <int L>
__host__ __device__ constexpr size_t cpre_doubles() { return (size_t)2 * ((1 << L) + L + 1); }

// Generic per-path walk (any per-step probabilities, any N, all kinds).
struct GenericArgs {
  double S0, K, u, d, disc, invN;
  double p[kMaxN];        // per-step up probabilities
  int N, g;               // 2^g codes per lane
  unsigned kinds;
  unsigned long long unit_first, unit_end;
  unsigned long long n_codes;  // 2^N (saturating for N = 64 is not needed: N <= 62)
};

struct Layout {
  int engine;   // 0 generic, 1 fast
  int L, D, m, Dp, g, q;
  unsigned long long units;
  int n_sb;
  unsigned long long units_per_sb;
};

}  // namespace bp

// C ABI of the binpaths B200 engine (include/binpaths_b200.h).
//
// Host side of the drop-in boundary: validation with the reference's error
// classes, layout selection, table construction, launches, multi-device
// sharding with one host thread per GPU, and the fixed-order combination of
// super-block partials.  Reference call sites: exact.py:75-133 (exact),
// mc.py:92-100,197-213,287-331 (Monte Carlo).
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <list>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <utility>
#include <vector>

#include "../../include/binpaths_b200.h"
#include "bp_exact.cuh"
#include "bp_kernels.h"
#include "bp_leaf.cuh"  // gray_table_entry (K1 shared-memory image)
#include "bp_threshold.h"
#include "bp_exact_w.cuh"

using namespace bp;

// ---------------------------------------------------------------------------
// error state
static thread_local std::string g_err;

static int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

#define BP_CUDA(call)                                                                          \
  do {                                                                                         \
    cudaError_t e_ = (call);                                                                   \
    if (e_ != cudaSuccess)                                                                     \
      return fail(BP_E_CUDA, std::string("CUDA error ") + cudaGetErrorString(e_) + " at " +    \
                                 __FILE__ + ":" + std::to_string(__LINE__) + " (" #call ")"); \
  } while (0)

extern "C" const char* bp_last_error(void) { return g_err.c_str(); }
extern "C" int bp_abi_version(void) { return BP_ABI_VERSION; }

extern "C" int bp_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

// ---------------------------------------------------------------------------
// validation (mirrors model.py:62-76 / exact.py:48-56 domains that the
// engine itself relies on; the Python mirror validates request objects
// before calling, so these are a second line of defence)
// any_sign_S0: the exact engine takes any finite S0, as the reference engine
// reads inputs.S0 unchecked (exact.py:96,99) -- the sign-flip oracle route of
// SURVEY 8(c); a non-positive S0 runs the per-path walk (choose_layout)
static int validate_tree(const bp_tree* t, int max_n, bool any_sign_S0 = false) {
  if (!t) return fail(BP_E_INVALID_INPUT, "tree is NULL");
  if (t->n_steps < 1 || t->n_steps > max_n)
    return fail(BP_E_INVALID_INPUT, "N must be between 1 and " + std::to_string(max_n) + ", got " +
                                        std::to_string(t->n_steps));
  if (!std::isfinite(t->S0)) return fail(BP_E_INVALID_INPUT, "S0 must be finite");
  if (!any_sign_S0 && !(t->S0 > 0.0)) return fail(BP_E_INVALID_INPUT, "S0 must be a positive finite number");
  if (!std::isfinite(t->K)) return fail(BP_E_INVALID_INPUT, "K must be finite");
  if (!(t->u > 0.0) || !std::isfinite(t->u) || !(t->d > 0.0) || !std::isfinite(t->d))
    return fail(BP_E_INVALID_INPUT, "u and d must be positive finite numbers");
  if (!std::isfinite(t->disc)) return fail(BP_E_INVALID_INPUT, "discount must be finite");
  if (!t->up_probs) return fail(BP_E_LENGTH_MISMATCH, "up_probs is NULL");
  for (int i = 0; i < t->n_steps; ++i) {
    const double p = t->up_probs[i];
    if (!(p >= 0.0 && p <= 1.0))
      return fail(BP_E_PROBABILITY, "up probability " + std::to_string(p) + " is outside [0, 1]");
  }
  return BP_OK;
}

static int kinds_ok(uint32_t payoffs) {
  if (payoffs == 0 || (payoffs >> BP_N_PAYOFFS) != 0)
    return fail(BP_E_INVALID_INPUT, "payoff mask must be a non-empty OR of bp_payoff bits");
  return BP_OK;
}

static bool constant_p(const bp_tree* t) {
  for (int i = 1; i < t->n_steps; ++i)
    if (t->up_probs[i] != t->up_probs[0]) return false;
  return true;
}

// ---------------------------------------------------------------------------
// layout: a pure function of (N, engine) so every device count and every
// machine uses the same decomposition (bitwise reproducibility across G).
// inner block bits of the fast engine (8 or 9; BINPATHS_INNER_BITS overrides)
// 9 since the I15 screen: its per-class work amortizes over bigger classes
// (config 2: 0.168 -> 0.146 ms, config 3: 4.12 -> 3.36 ms); 10 was measured
// slower (0.232 / 6.2 ms: the unrolled classes outgrow the instruction cache;
// profiles/r2_scan_inner_bits.log)
static int fast_L() {
  static int L = [] {
    const char* e = std::getenv("BINPATHS_INNER_BITS");
    const int v = e ? std::atoi(e) : 9;
    return (v == 8 || v == 9) ? v : 9;
  }();
  return L;
}

static void build_inner(int L, double u, double d, std::vector<double>& c, std::vector<double>& mx,
                        std::vector<double>& mn, std::vector<double>& e, std::vector<int>& h) {
  const int n = 1 << L;
  c.assign(n, 0.0);
  mx.assign(n, 0.0);
  mn.assign(n, 0.0);
  e.assign(n, 1.0);
  h.assign(n, 0);
  for (int s = 0; s < n; ++s) {
    double r = 1.0, cs = 0.0, m1 = 0.0, m2 = INFINITY;
    int ups = 0;
    for (int j = 0; j < L; ++j) {
      const int b = (s >> (L - 1 - j)) & 1;
      r *= b ? u : d;
      cs += r;
      m1 = std::max(m1, r);
      m2 = std::min(m2, r);
      ups += b;
    }
    c[s] = cs;
    mx[s] = m1;
    mn[s] = m2;
    e[s] = r;
    h[s] = ups;
  }
}

static Layout choose_layout(const bp_tree* t, uint32_t payoffs, uint32_t flags, bool* fast_possible) {
  const int N = t->n_steps;
  Layout lay{};
  const bool pos = t->S0 > 0.0;  // the class engines divide by the node price
  if ((flags & BP_FLAG_THRESHOLD) && pos && N >= kFastMinN && constant_p(t) && t->up_probs[0] > 0.0 &&
      t->up_probs[0] < 1.0 && t->u > t->d) {
    // K8 threshold search: 2^LT leaves per node, >= 2^16 nodes when N allows
    lay.engine = 2;
    lay.L = std::max(8, std::min(20, N - 16));
    lay.D = N - lay.L;
    lay.m = 0;
    lay.Dp = lay.D;
    const int free_bits = lay.D - 5;
    lay.q = std::max(0, free_bits - 18);
    lay.units = 1ull << (free_bits - lay.q);
    lay.g = 0;
    lay.n_sb = (int)std::min<unsigned long long>(kMaxSB, lay.units);
    lay.units_per_sb = lay.units / lay.n_sb;
    if (fast_possible) *fast_possible = false;
    return lay;
  }
  static const bool force_w = [] {
    const char* e = std::getenv("BINPATHS_WEIGHTED");
    return e && std::atoi(e) != 0;
  }();
  // K1w: per-leaf weights (any per-step probabilities) -- the explicit engine
  // for non-constant p, and for constant p when BINPATHS_WEIGHTED=1
  // (leaf bookkeeping is not implemented in K1w: BP_FLAG_COUNT takes the path walk)
  if (!(flags & (BP_FLAG_GENERIC | BP_FLAG_COUNT)) && pos && N >= kFastMinN && t->u > t->d &&
      (force_w || !constant_p(t))) {
    lay.engine = 3;
    lay.L = 8;
    lay.D = N - lay.L;
    const int free_bits = lay.D - 5;
    lay.m = std::max(2, std::min(6, free_bits - kUnitTargetLog2));  // >= 2: nodes go in fours
    lay.Dp = lay.D - lay.m;
    const int unit_bits = std::max(0, free_bits - lay.m);
    lay.q = std::max(0, unit_bits - 18);
    lay.units = 1ull << (unit_bits - lay.q);
    lay.g = 0;
    lay.n_sb = (int)std::min<unsigned long long>(kMaxSB, lay.units);
    lay.units_per_sb = lay.units / lay.n_sb;
    if (fast_possible) *fast_possible = true;
    return lay;
  }
  bool fast = !(flags & BP_FLAG_GENERIC) && pos && N >= kFastMinN && constant_p(t);
  if (fast) {
    const double p = t->up_probs[0];
    if (!(p > 0.0 && p < 1.0)) fast = false;  // degenerate: single-path mass, walk it
  }
  if (fast) {
    // every requested kind must have a fast kernel (each kind can be launched alone)
    for (int k = 0; k < kNumKinds; ++k)
      if (((payoffs >> k) & 1) && !fast_kind_mask_supported(1u << k)) fast = false;
  }
  if (fast) {
    // every inner-table entry is a sum of L products of at most L factors u or
    // d, so all are finite iff L * max(u, d, 1)^L is
    const double big = std::max(1.0, std::max(t->u, t->d));
    if (!std::isfinite(std::pow(big, fast_L()) * fast_L())) fast = false;
  }
  if (fast_possible) *fast_possible = fast;
  if (fast) {
    lay.engine = 1;
    lay.L = fast_L();
    lay.D = N - lay.L;
    const int free_bits = lay.D - 5;  // bits above the lane
    static const int target = [] {
      const char* e = std::getenv("BINPATHS_UNIT_LOG2");
      return e ? std::atoi(e) : kFastUnitTargetLog2;
    }();
    // n_mid = 2^m is a multiple of the nodes per leaf block; at most 2^kMidCap
    // nodes per lane per unit keeps >= ~14 units per warp at 8 ranks for the
    // N = 36 tree (wave quantization), at ~1 % more prefix walks
    static const int mid_cap = [] {
      const char* e = std::getenv("BINPATHS_MID_CAP");  // diagnostics
      const int v = e ? std::atoi(e) : kMidCap;
      return (v >= 1 && v <= 6) ? v : kMidCap;
    }();
    lay.m = std::max(std::max(1, kNodesPerBlockLog2), std::min(mid_cap, free_bits - target));
    lay.Dp = lay.D - lay.m;
    const int unit_bits = free_bits - lay.m;
    lay.q = std::max(0, unit_bits - 18);
    lay.units = 1ull << (unit_bits - lay.q);
    lay.g = 0;
  } else {
    lay.engine = 0;
    lay.L = 0;
    lay.D = N;
    const int free_bits = std::max(0, N - 5);
    lay.g = std::max(0, free_bits - kUnitTargetLog2);
    lay.units = 1ull << (free_bits - lay.g);
    lay.m = lay.Dp = lay.q = 0;
  }
  lay.n_sb = (int)std::min<unsigned long long>(kMaxSB, lay.units);
  lay.units_per_sb = lay.units / lay.n_sb;
  return lay;
}

// Inner table of one kind, laid out by position: class-major, sorted inside a
// class in the kind's compare direction (descending for '>' kinds AC / FL,
// ascending for '<' kinds AP / FLP), plus the group prefix sums.
template <int L>
static void kind_table_layout(int kind, const std::vector<double>& c, const std::vector<double>& mx,
                              const std::vector<double>& mn, double* pos_out /* 2^L */,
                              double (*gpre)[kGroupSlots] /* n_groups(L) */) {
  const std::vector<double>& v = (kind == kAC || kind == kAP) ? c : (kind == kFL) ? mx : mn;
  const bool desc = (kind == kAC || kind == kFL);
  for (int cl = 0; cl <= L; ++cl) {
    std::vector<double> cls;
    for (int s = 0; s < (1 << L); ++s)
      if (__builtin_popcount((unsigned)s) == cl) cls.push_back(v[s]);
    if (desc)
      std::sort(cls.begin(), cls.end(), [](double a, double b) { return a > b; });
    else
      std::sort(cls.begin(), cls.end());
    const int start = class_start(L, cl);
    for (size_t i = 0; i < cls.size(); ++i) pos_out[start + i] = cls[i];
    for (int g = 0; g < class_groups(L, cl); ++g) {
      double* P = gpre[group_base(L, cl) + g];
      const int len = std::min<int>(kGroup, (int)cls.size() - kGroup * g);
      double sum = 0.0, comp = 0.0;  // compensated prefix sums, rounded once
      P[0] = 0.0;
      for (int n = 1; n < kGroupSlots; ++n) {
        if (n <= len) comp_add(sum, comp, cls[kGroup * g + n - 1]);
        P[n] = sum + comp;
      }
    }
  }
}

// I15 screen tables of one slot (bp_exact.cuh, bp_leaf.cuh I15Class): per big
// class a monotone map onto [0, 32767] spanning the class's values
// (increasing for '>' kinds, decreasing for '<' kinds, so that in both cases
// a screened value above the threshold's proves the leaf in the money), the
// screened value of every position in both 16-bit lanes, and the class
// prefix sums in sorted order (compensated, rounded once).
template <int L>
static void i15_layout(int kind, const double* pos, ExactArgs<L>& a, ExactTables<L>& tb, int slot) {
  const bool desc = (kind == kAC || kind == kFL);
  for (int c = 0; c <= L; ++c) {
    a.nrm_s[slot][c] = 1.0f;
    a.nrm_o[slot][c] = kI15Magic;
    if (!i15_class(L, c)) continue;
    const int i0 = class_start(L, c), len = binom(L, c);
    float lo = (float)pos[i0], hi = (float)pos[i0];
    for (int j = 0; j < len; ++j) {
      lo = std::min(lo, (float)pos[i0 + j]);
      hi = std::max(hi, (float)pos[i0 + j]);
    }
    // the class spans the codes [4, 32763]: a clamped threshold (0 or
    // 32767) never equals a screened value; |v s| <= 2^22 keeps the fp32
    // products resolved to half a code
    const float range = hi - lo, amax = std::max(std::fabs(lo), std::fabs(hi));
    double sc = range > 0.0f ? 32759.0 / (double)range : 1.0;
    if (amax > 0.0f) sc = std::min(sc, 4194304.0 / (double)amax);
    if (!(sc > 0.0) || !std::isfinite(sc)) sc = 1.0;
    const float sf = (float)(desc ? sc : -sc);
    // the end of the range the map sends to code 4
    const double o = (double)kI15Magic + 4.0 - (double)(desc ? lo : hi) * (double)sf;
    a.nrm_s[slot][c] = sf;
    a.nrm_o[slot][c] = std::isfinite(o) ? (float)o : kI15Magic;
    for (int j = 0; j < len; ++j) {
      int e = j + 1;
      const double tol = std::ldexp(std::fabs(pos[i0 + j]), -44);
      while (e < len && std::fabs(pos[i0 + e] - pos[i0 + j]) <= tol) ++e;
      tb.te[slot][i0 + j] = (unsigned char)e;
    }
    double sum = 0.0, comp = 0.0;
    tb.cpre[slot][i0 + c] = 0.0;
    for (int j = 0; j < len; ++j) {
      const unsigned k = i15_map((float)pos[i0 + j], a.nrm_s[slot][c], a.nrm_o[slot][c]);
      tb.xq[slot][i0 + j] = k | (k << 16);
      comp_add(sum, comp, pos[i0 + j]);
      tb.cpre[slot][i0 + c + j + 1] = sum + comp;
    }
  }
}

// the screen tables of one slot of a host argument block (i15_quarter)
template <int L>
struct HostTabs {
  const ExactArgs<L>& a;
  const ExactTables<L>& tb;
  int slot;
  __host__ __device__ double tab(int i) const { return a.tab[slot * (1 << L) + i]; }
  __host__ __device__ double cpre(int i) const { return tb.cpre[slot][i]; }
  __host__ __device__ unsigned xq(int i) const { return tb.xq[slot][i]; }
  __host__ __device__ unsigned te(int i) const { return tb.te[slot][i]; }
};

// K1's shared-memory image (k1_smem_layout), appended to the argument block:
// the tables every CTA used to build from the parameter bank, built once here
// with the same formulas (kernel fallback: bp_exact_fast.cuh, ga == nullptr).
template <int L>
static void build_smem_image(const ExactArgs<L>& a, const ExactTables<L>& tb, unsigned km, unsigned char* img) {
  const K1SmemLayout ly = k1_smem_layout<L>(km);
  std::memset(img, 0, ly.total);
  constexpr int NC = L + 1, NG = n_groups(L);
  double* sw = reinterpret_cast<double*>(img + ly.sw);
  for (int i = 0; i < kMaxN + 2 + NC; ++i) sw[i] = i < kMaxN + 2 ? a.w[i] : 0.0;
  if (ly.need_w) {
    double* w1 = reinterpret_cast<double*>(img + ly.sW1);
    double* w2 = reinterpret_cast<double*>(img + ly.sW2);
    for (int i = 0; i < kMaxN + 2; ++i) {
      double s1 = 0.0, s2 = 0.0;
      for (int c = 0; c < NC; ++c) {
        s1 = std::fma(sw[i + c], a.b_cls[c], s1);
        s2 = std::fma(sw[i + c] * a.b_cls[c], a.e_cls[c], s2);
      }
      w1[i] = s1;
      w2[i] = s2;
    }
  }
  auto gray_groups = [&](int slot, double2* dst, bool small_only) {
    int k = 0;
    for (int c = 0; c <= L; ++c) {
      if (small_only && i15_class(L, c)) continue;
      for (int g = 0; g < class_groups(L, c); ++g, ++k)
        for (int sl = 0; sl < kGraySlots; ++sl)
          dst[k * kGraySlots + sl] = gray_table_entry(&tb.gpre[slot][group_base(L, c) + g][0], (unsigned)sl, true);
    }
    (void)NG;
  };
  for (int slot = 0; slot < ly.nt && slot < 2; ++slot) {
    gray_groups(slot, reinterpret_cast<double2*>(img + ly.sgray[slot]), ly.i15[slot]);
    if (!ly.i15[slot]) continue;
    double2* et = reinterpret_cast<double2*>(img + ly.si15[slot]);
    const HostTabs<L> ht{a, tb, slot};
    for (int c = 0; c <= L; ++c) {
      if (!i15_class(L, c)) continue;
      const int len = binom(L, c), i0 = class_start(L, c), base = i15_base(L, c), slots = i15_slots(L, c);
      const int nq = i15_entry_bytes(ly.lookback[slot]) / 16;
      for (int t = 0; t < nq * slots; ++t) {
        unsigned n = (unsigned)(t / nq);
        for (int sh = 1; sh < 16; sh <<= 1) n ^= n >> sh;  // Gray -> binary
        et[nq * base + t] = i15_quarter(ht, c, i0, len, (int)n, t % nq, ly.lookback[slot]);
      }
    }
    std::memcpy(img + ly.sxq[slot], tb.xq[slot], sizeof(unsigned) << L);
    std::memcpy(img + ly.ste[slot], tb.te[slot], (size_t)1 << L);
  }
}

template <int L>
static int fill_fast_args(const bp_tree* t, const Layout& lay, unsigned km, std::vector<unsigned char>& buf) {
  buf.assign(sizeof(ExactArgs<L>), 0);
  ExactArgs<L>& a = *reinterpret_cast<ExactArgs<L>*>(buf.data());
  auto tables = std::make_unique<ExactTables<L>>();  // setup-only tables (device image)
  ExactTables<L>& tbl = *tables;
  std::memset(&tbl, 0, sizeof(tbl));
  std::vector<double> c, mx, mn, e;
  std::vector<int> h;
  build_inner(L, t->u, t->d, c, mx, mn, e, h);
  // table slots in kind order AC, AP, FL, FLP (must match k_exact_fast)
  std::vector<int> kinds;
  for (int k : {kAC, kAP, kFL, kFLP})
    if ((km >> k) & 1) kinds.push_back(k);
  if (kinds.size() > 2) return fail(BP_E_INVALID_INPUT, "more than two inner tables requested in one launch");
  const int nt = (int)kinds.size();
  std::vector<double> pos(1 << L);
  for (int slot = 0; slot < nt; ++slot) {
    kind_table_layout<L>(kinds[slot], c, mx, mn, pos.data(), tbl.gpre[slot]);
    for (int i = 0; i < (1 << L); ++i) a.tab[slot * (1 << L) + i] = pos[i];
    if constexpr (i15_on<L>()) i15_layout<L>(kinds[slot], pos.data(), a, tbl, slot);
  }
  // middle tables (chunk of m steps)
  const int m = lay.m;
  std::vector<double> mc, mmx, mmn, me;
  std::vector<int> mh;
  if (m > 0) {
    build_inner(m, t->u, t->d, mc, mmx, mmn, me, mh);
  } else {
    mc = {0.0};
    mmx = {0.0};
    mmn = {INFINITY};
    me = {1.0};
    mh = {0};
  }
  for (int j = 0; j < (1 << m); ++j) {
    a.mid_c[j] = mc[j];
    a.mid_e[j] = me[j];
    a.mid_mx[j] = mmx[j];
    a.mid_mn[j] = mmn[j];
    a.mid_h[j] = mh[j];
  }
  // weights, discount folded in (exact.py:95,99)
  const int N = t->n_steps;
  const double p = t->up_probs[0];
  for (int k = 0; k <= N; ++k) a.w[k] = t->disc * std::pow(p, k) * std::pow(1.0 - p, N - k);
  for (int k = N + 1; k < kMaxN + 2; ++k) a.w[k] = 0.0;
  for (int cc = 0; cc <= L; ++cc) {
    double r = 1.0;
    for (int j = 0; j < cc; ++j) r *= t->u;
    for (int j = cc; j < L; ++j) r *= t->d;
    a.e_cls[cc] = r;
    a.b_cls[cc] = (double)binom(L, cc);
  }
  ExactScalars& s = a.s;
  s.S0 = t->S0;
  s.K = t->K;
  s.NK = (double)N * t->K;
  s.u = t->u;
  s.d = t->d;
  s.invN = 1.0 / N;
  s.N = N;
  s.L = L;
  s.D = lay.D;
  s.m = m;
  s.Dp = lay.Dp;
  s.n_mid = 1 << m;
  s.q = lay.q;
  s.zero = 0;
  // the device image after the block: the shared-memory image (K1's CTA
  // setup copies it), then the class prefix sums (the exact walk reads them)
  const size_t head = align16(sizeof(ExactArgs<L>));
  const size_t simg = k1_smem_layout<L>(km).total;
  buf.resize(head + simg + sizeof(double) * cpre_doubles<L>(), 0);
  build_smem_image<L>(*reinterpret_cast<ExactArgs<L>*>(buf.data()), tbl, km, buf.data() + head);
  std::memcpy(buf.data() + head + simg, &tbl.cpre[0][0], sizeof(double) * cpre_doubles<L>());
  return BP_OK;
}

// K1w arguments: per-step weights, one sorted table per kind + group prefix sums
static int fill_w_args(const bp_tree* t, const Layout& lay, unsigned km, std::vector<unsigned char>& buf) {
  constexpr int L = 8, NL = 1 << L, NG = NL / kWGroup;
  buf.assign(sizeof(ExactWArgs<L>), 0);
  ExactWArgs<L>& a = *reinterpret_cast<ExactWArgs<L>*>(buf.data());
  const int N = t->n_steps, D = lay.D, m = lay.m, Dp = lay.Dp;
  std::vector<double> c, mx, mn, e;
  std::vector<int> h;
  build_inner(L, t->u, t->d, c, mx, mn, e, h);
  // inner weights: steps D .. N-1 (0-based), step D = most significant bit of s
  std::vector<double> w(NL, 1.0);
  for (int s2 = 0; s2 < NL; ++s2)
    for (int j = 0; j < L; ++j) {
      const double p = t->up_probs[D + j];
      w[s2] *= ((s2 >> (L - 1 - j)) & 1) ? p : 1.0 - p;
    }
  std::vector<int> kinds;
  for (int k = 0; k < kNumKinds; ++k)  // slot order = kind-bit order (k_exact_w)
    if ((km >> k) & 1) kinds.push_back(k);
  if (kinds.size() > 2) return fail(BP_E_INVALID_INPUT, "more than two kinds in one launch");
  for (size_t slot = 0; slot < kinds.size(); ++slot) {
    const int k = kinds[slot];
    const std::vector<double>& v = (k == kAC || k == kAP) ? c : (k == kFL) ? mx : (k == kFLP) ? mn : e;
    const bool desc = (k == kAC || k == kFL || k == kEC);
    std::vector<int> ord(NL);
    for (int i = 0; i < NL; ++i) ord[i] = i;
    std::stable_sort(ord.begin(), ord.end(), [&](int x, int y) { return desc ? v[x] > v[y] : v[x] < v[y]; });
    for (int i = 0; i < NL; ++i) a.tab[slot * NL + i] = v[ord[i]];
    for (int g = 0; g < NG; ++g) {
      double sa = 0.0, ca = 0.0, sb = 0.0, cb = 0.0;
      a.gp[slot][g * (kWGroup + 1)] = make_double2(0.0, 0.0);
      for (int n = 1; n <= kWGroup; ++n) {
        const int s2 = ord[kWGroup * g + n - 1];
        comp_add(sa, ca, w[s2] * v[s2]);
        comp_add(sb, cb, w[s2]);
        a.gp[slot][g * (kWGroup + 1) + n] = make_double2(sa + ca, sb + cb);
      }
    }
  }
  double E = 0.0, Ec = 0.0, O = 0.0, Oc = 0.0;
  for (int s2 = 0; s2 < NL; ++s2) {
    comp_add(E, Ec, w[s2] * e[s2]);
    comp_add(O, Oc, w[s2]);
  }
  // middle tables (steps Dp .. D-1)
  for (int j = 0; j < (1 << m); ++j) {
    double r = 1.0, cs = 0.0, m1 = 0.0, m2 = INFINITY, ww = 1.0;
    for (int i = 0; i < m; ++i) {
      const int b = (j >> (m - 1 - i)) & 1;
      const double p = t->up_probs[Dp + i];
      r *= b ? t->u : t->d;
      cs += r;
      m1 = std::max(m1, r);
      m2 = std::min(m2, r);
      ww *= b ? p : 1.0 - p;
    }
    a.mid_c[j] = cs;
    a.mid_e[j] = r;
    a.mid_mx[j] = m1;
    a.mid_mn[j] = m2;
    a.mid_w[j] = ww;
  }
  for (int i = 0; i < Dp; ++i) {
    a.p[i] = t->up_probs[i];
    a.q[i] = 1.0 - t->up_probs[i];
  }
  ExactWScalars& sc = a.s;
  sc.S0 = t->S0;
  sc.K = t->K;
  sc.NK = (double)N * t->K;
  sc.u = t->u;
  sc.d = t->d;
  sc.disc = t->disc;
  sc.E = E + Ec;
  sc.Omega = O + Oc;
  sc.N = N;
  sc.L = L;
  sc.D = D;
  sc.m = m;
  sc.Dp = Dp;
  sc.n_mid = 1 << m;
  sc.q = lay.q;
  sc.zero = 0;
  return BP_OK;
}

// K1 arguments depend on the contract (S0, K) only through three scalars;
// the tables (class-sorted inner tables, group prefix sums, middle tables,
// weights) are a function of the lattice.  A small LRU of built argument
// blocks keyed by the lattice makes revaluing on a known lattice (new spot or
// strike, or the same contract again) skip the host table build (~20 us).
struct FastArgsKey {
  int L, D, m, Dp, q, N;
  unsigned km;
  double u, d, p, disc;
  bool operator==(const FastArgsKey& o) const {
    return L == o.L && D == o.D && m == o.m && Dp == o.Dp && q == o.q && N == o.N && km == o.km && u == o.u &&
           d == o.d && p == o.p && disc == o.disc;
  }
};

// the scalars of an argument block of inner block size L
static ExactScalars* exact_scalars(std::vector<unsigned char>& buf, int L) {
  return L == 8 ? &reinterpret_cast<ExactArgs<8>*>(buf.data())->s : &reinterpret_cast<ExactArgs<9>*>(buf.data())->s;
}

static void set_contract(std::vector<unsigned char>& buf, int L, const bp_tree* t) {
  ExactScalars* s = exact_scalars(buf, L);
  s->S0 = t->S0;
  s->K = t->K;
  s->NK = (double)t->n_steps * t->K;
}

static int build_fast_args(const bp_tree* t, const Layout& lay, unsigned km, std::vector<unsigned char>& buf,
                           FastArgsKey* key_out = nullptr) {
  static std::mutex mu;
  static std::list<std::pair<FastArgsKey, std::vector<unsigned char>>> lru;  // most recent first
  constexpr size_t kCap = 16;
  const FastArgsKey key{lay.L, lay.D, lay.m, lay.Dp, lay.q, t->n_steps, km, t->u, t->d, t->up_probs[0], t->disc};
  if (key_out) *key_out = key;
  {
    std::lock_guard<std::mutex> g(mu);
    for (auto it = lru.begin(); it != lru.end(); ++it)
      if (it->first == key) {
        lru.splice(lru.begin(), lru, it);
        buf = it->second;
        set_contract(buf, lay.L, t);
        return BP_OK;
      }
  }
  int rc;
  switch (lay.L) {
    case 8: rc = fill_fast_args<8>(t, lay, km, buf); break;
    case 9: rc = fill_fast_args<9>(t, lay, km, buf); break;
    default: return fail(BP_E_INVALID_INPUT, "unsupported inner block size");
  }
  if (rc) return rc;
  std::lock_guard<std::mutex> g(mu);
  lru.emplace_front(key, buf);
  if (lru.size() > kCap) lru.pop_back();
  return BP_OK;
}

// Device images of K1 argument blocks (the tables K1's CTA setup reads;
// k_exact_fast's `ga`), per device, keyed by lattice + layout + kinds.  Kept
// for the life of the process (graphs captured with them stay valid), at most
// kMaxImages per device; beyond that a plan uploads (and frees) its own.
struct DevArgImage {
  FastArgsKey key;
  void* p;
};
static std::mutex g_img_mu;
static std::vector<DevArgImage> g_img[64];
constexpr size_t kMaxImages = 256;

// the device's cached image for key (uploaded on first use), or nullptr when
// the cache is full.  Not callable inside a stream capture.
static void* cached_arg_image(int dev, const FastArgsKey& key, const std::vector<unsigned char>& args) {
  std::lock_guard<std::mutex> g(g_img_mu);
  for (auto& im : g_img[dev])
    if (im.key == key) return im.p;
  if (g_img[dev].size() >= kMaxImages) return nullptr;
  void* p = nullptr;
  if (cudaMalloc(&p, args.size()) != cudaSuccess) return nullptr;
  if (cudaMemcpy(p, args.data(), args.size(), cudaMemcpyHostToDevice) != cudaSuccess) {
    cudaFree(p);
    return nullptr;
  }
  g_img[dev].push_back(DevArgImage{key, p});
  return p;
}

static void set_units_w(std::vector<unsigned char>& buf, unsigned long long u0, unsigned long long u1) {
  ExactWScalars* s = &reinterpret_cast<ExactWArgs<8>*>(buf.data())->s;
  s->unit_first = u0;
  s->unit_end = u1;
}

static void set_units(std::vector<unsigned char>& buf, int L, unsigned long long u0, unsigned long long u1) {
  ExactScalars* s = exact_scalars(buf, L);
  s->unit_first = u0;
  s->unit_end = u1;
}

// the groups of kinds launched together in the fast engine
static std::vector<unsigned> fast_groups(uint32_t payoffs) {
  std::vector<unsigned> g;
  unsigned rest = payoffs;
  const unsigned pair = (1u << kAC) | (1u << kFL);
  static const bool fuse = [] {  // diagnostics: BINPATHS_FUSE_ACFL=0 launches the pair apart
    const char* e = std::getenv("BINPATHS_FUSE_ACFL");
    return !e || std::atoi(e) != 0;
  }();
  if (fuse && (rest & pair) == pair) {
    g.push_back(pair);
    rest &= ~pair;
  }
  for (int k = 0; k < kNumKinds; ++k)
    if ((rest >> k) & 1) g.push_back(1u << k);
  return g;
}

// keep freed stream-ordered allocations in the device pool (scratch is
// re-allocated every valuation; returning it to the OS costs milliseconds)
static void keep_pool(int dev) {
  static std::mutex mu;
  static bool done[64] = {false};
  std::lock_guard<std::mutex> g(mu);
  if (dev < 0 || dev >= 64 || done[dev]) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    uint64_t thr = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  done[dev] = true;
}

// occupancy of a K1 instantiation (a property of the compiled kernel and the
// device type; queried once)
static int cached_occupancy_fast(int L, unsigned km, bool cnt) {
  static std::mutex mu;
  static std::vector<std::pair<unsigned, int>> memo;
  const unsigned key = ((unsigned)L << 16) | (km << 1) | (cnt ? 1u : 0u);
  std::lock_guard<std::mutex> g(mu);
  for (auto& e : memo)
    if (e.first == key) return e.second;
  const int occ = occupancy_exact_fast(L, km, cnt);
  memo.emplace_back(key, occ);
  return occ;
}

// BINPATHS_TRACE=1: host-side phase timings on stderr (diagnostics)
static bool trace_on() {
  static const bool on = [] {
    const char* e = std::getenv("BINPATHS_TRACE");
    return e && std::atoi(e) != 0;
  }();
  return on;
}

static int device_sm_count(int dev) {
  static std::atomic<int> memo[64];
  if (dev >= 0 && dev < 64 && memo[dev].load() > 0) return memo[dev].load();
  int n = 0;
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  if (n > 0 && dev >= 0 && dev < 64) memo[dev].store(n);
  return n > 0 ? n : 1;
}

// Enqueue the valuation of super-blocks [sb_first, sb_first+sb_count) on
// the current device.  out_dev: [sb_count][6][2] doubles (device).
// Unit scratch of a valuation: a head of kScratchHead double2 (slot 0 = K1's
// unit counter, 0 between launches: zeroed at allocation, reset by the K2
// after every K1), then the unit partials [unit][kind].
constexpr size_t kScratchHead = 16;
static size_t scratch_need(unsigned long long n_units) {
  return sizeof(double2) * (kScratchHead + (size_t)kNumKinds * n_units);
}
static cudaError_t scratch_alloc(double2** p, size_t bytes, cudaStream_t st) {
  cudaError_t e = cudaMallocAsync((void**)p, bytes, st);
  if (e == cudaSuccess) e = cudaMemsetAsync(*p, 0, sizeof(double2) * kScratchHead, st);
  return e;
}

// ---------------------------------------------------------------------------
// A prepared valuation: layout, prebuilt kernel arguments per kind group and
// per-device scratch.  Building the tables costs host time (sorting, pow);
// a plan does it once so repeated launches are launches only.
struct bp_exact_plan {
  bp_tree tree;
  std::vector<double> probs;
  uint32_t payoffs = 0, flags = 0;
  Layout lay{};
  struct Group {
    unsigned km;
    std::vector<unsigned char> args;
    FastArgsKey key{};           // class engine: the lattice key of args
    void* dargs[64] = {nullptr};  // class engine: device image per device
    bool dargs_owned[64] = {false};
  };
  std::vector<Group> groups;
  GenericArgs gen{};
  // K8 tables (host copies; uploaded per device on first use)
  std::vector<double> th_tables;  // [slot][val 2^LT | pre 2^LT + LT + 1]
  int th_nt = 0;
  ThresholdArgs th{};
  double* th_dev[64] = {nullptr};
  struct Scratch {
    double2* p = nullptr;
    size_t bytes = 0;
  };
  Scratch scratch[64];
  std::mutex mu;
  // captured enqueues of the class engine, keyed by (device, super-block
  // range, output buffer, scratch): a repeated enqueue is one graph launch.
  // A key is captured the second time it is seen in a row (a caller with a
  // fresh output buffer per call keeps the ordinary launches), and at most
  // kMaxPlanGraphs stay instantiated (least recently used out first).
  struct Graph {
    int dev, sb_first, sb_count;
    double* out;
    double2* scratch;
    cudaGraphExec_t exec;
    bool same(const Graph& o) const {
      return dev == o.dev && sb_first == o.sb_first && sb_count == o.sb_count && out == o.out &&
             scratch == o.scratch;
    }
  };
  static constexpr size_t kMaxPlanGraphs = 8;
  std::list<Graph> graphs;
  Graph last_miss{-1, 0, 0, nullptr, nullptr, nullptr};
};

static int plan_build(const bp_tree* t, uint32_t payoffs, uint32_t flags, bp_exact_plan* P) {
  P->probs.assign(t->up_probs, t->up_probs + t->n_steps);
  P->tree = *t;
  P->tree.up_probs = P->probs.data();
  P->payoffs = payoffs;
  P->flags = flags;
  P->lay = choose_layout(t, payoffs, flags, nullptr);
  const Layout& lay = P->lay;
  if (lay.engine == 3) {
    for (unsigned km : fast_groups(payoffs)) {
      bp_exact_plan::Group g;
      g.km = km;
      int rc = fill_w_args(&P->tree, lay, km, g.args);
      if (rc) return rc;
      P->groups.push_back(std::move(g));
    }
  } else if (lay.engine == 1) {
    for (unsigned km : fast_groups(payoffs)) {
      bp_exact_plan::Group g;
      g.km = km;
      int rc = build_fast_args(&P->tree, lay, km, g.args, &g.key);
      if (rc) return rc;
      P->groups.push_back(std::move(g));
    }
  } else if (lay.engine == 2) {
    const int LT = lay.L, NL = 1 << LT;
    std::vector<double> c, mx, mn, e;
    std::vector<int> h;
    build_inner(LT, t->u, t->d, c, mx, mn, e, h);
    ThresholdArgs& a = P->th;
    // classes in popcount order: offsets, and the per-leaf position
    std::vector<int> off(LT + 2, 0);
    for (int cl = 0; cl <= LT; ++cl) off[cl + 1] = off[cl] + binom(LT, cl);
    for (int cl = 0; cl <= LT + 1; ++cl) a.class_off[cl] = off[cl];
    const size_t slot_sz = (size_t)NL + NL + LT + 1;
    // kind slots in kind-bit order (k_exact_threshold walks k = 0..5)
    std::vector<int> kinds;
    for (int k = 0; k < kNumKinds; ++k)
      if (((payoffs >> k) & 1) && k != kEC && k != kEP) kinds.push_back(k);
    P->th_nt = (int)kinds.size();
    P->th_tables.assign(slot_sz * std::max(1, P->th_nt), 0.0);
    std::vector<std::vector<double>> cls(LT + 1);
    for (int slot = 0; slot < P->th_nt; ++slot) {
      const int k = kinds[slot];
      const std::vector<double>& v = (k == kAC || k == kAP) ? c : (k == kFL) ? mx : mn;
      const bool desc = (k == kAC || k == kFL);
      for (auto& x : cls) x.clear();
      for (int s2 = 0; s2 < NL; ++s2) cls[__builtin_popcount((unsigned)s2)].push_back(v[s2]);
      double* val = P->th_tables.data() + slot * slot_sz;
      double* pre = val + NL;
      for (int cl = 0; cl <= LT; ++cl) {
        auto& x = cls[cl];
        if (desc)
          std::sort(x.begin(), x.end(), [](double p1, double p2) { return p1 > p2; });
        else
          std::sort(x.begin(), x.end());
        double sum = 0.0, comp = 0.0;
        pre[off[cl] + cl] = 0.0;
        for (size_t i = 0; i < x.size(); ++i) {
          val[off[cl] + i] = x[i];
          comp_add(sum, comp, x[i]);
          pre[off[cl] + cl + i + 1] = sum + comp;
        }
      }
    }
    const int N = t->n_steps;
    const double p = t->up_probs[0];
    for (int k = 0; k < kMaxN + 2 + kMaxThreshL + 1; ++k)
      a.w[k] = (k <= N) ? t->disc * std::pow(p, k) * std::pow(1.0 - p, N - k) : 0.0;
    for (int cc = 0; cc <= LT; ++cc) {
      double r = 1.0;
      for (int j = 0; j < cc; ++j) r *= t->u;
      for (int j = cc; j < LT; ++j) r *= t->d;
      a.e_cls[cc] = r;
      a.b_cls[cc] = (double)binom(LT, cc);
    }
    a.S0 = t->S0;
    a.K = t->K;
    a.NK = (double)N * t->K;
    a.u = t->u;
    a.d = t->d;
    a.N = N;
    a.LT = LT;
    a.D = lay.D;
    a.m = 0;
    a.Dp = lay.D;
    a.q = lay.q;
    a.kinds = payoffs;
  } else {
    GenericArgs& g = P->gen;
    g.S0 = t->S0;
    g.K = t->K;
    g.u = t->u;
    g.d = t->d;
    g.disc = t->disc;
    g.invN = 1.0 / t->n_steps;
    for (int i = 0; i < t->n_steps; ++i) g.p[i] = t->up_probs[i];
    g.N = t->n_steps;
    g.g = lay.g;
    g.kinds = payoffs;
    g.n_codes = 1ull << t->n_steps;
  }
  return BP_OK;
}

// Enqueue the valuation of super-blocks [sb_first, sb_first+sb_count) on
// device `dev` (current).  out_dev: [sb_count][6][2] doubles (device).
// The plan's scratch for `dev` is reused: calls on one plan and device must
// be issued on one stream (stream order protects the reuse).
static int plan_attach_images(bp_exact_plan* P, int dev, cudaStream_t st);

static int plan_enqueue(bp_exact_plan* P, int dev, int sb_first, int sb_count, double* out_dev,
                        unsigned long long* hist_dev, cudaStream_t st) {
  const Layout& lay = P->lay;
  if (dev >= 0 && dev < 64) {
    const int rc = plan_attach_images(P, dev, st);  // a no-op once attached (always so inside captures)
    if (rc) return rc;
  }
  if (sb_first < 0 || sb_count < 1 || sb_first + sb_count > lay.n_sb)
    return fail(BP_E_RANK_RANGE, "super-block range [" + std::to_string(sb_first) + ", " +
                                     std::to_string(sb_first + sb_count) + ") outside [0, " +
                                     std::to_string(lay.n_sb) + ")");
  if (dev < 0 || dev >= 64) return fail(BP_E_NO_DEVICE, "device index out of range");
  const bool cnt = (P->flags & BP_FLAG_COUNT) != 0;
  if (cnt && !hist_dev) return fail(BP_E_INVALID_INPUT, "BP_FLAG_COUNT needs a histogram buffer");
  const unsigned long long u0 = (unsigned long long)sb_first * lay.units_per_sb;
  const unsigned long long u1 = u0 + (unsigned long long)sb_count * lay.units_per_sb;
  const unsigned long long n_units = u1 - u0;
  double2* unit_out = nullptr;
  unsigned long long* work = nullptr;
  {
    std::lock_guard<std::mutex> g(P->mu);
    auto& sc = P->scratch[dev];
    const size_t need = scratch_need(n_units);
    if (sc.bytes < need) {
      if (sc.p) cudaFreeAsync(sc.p, st);
      sc.p = nullptr;
      sc.bytes = 0;
      BP_CUDA(scratch_alloc(&sc.p, need, st));
      sc.bytes = need;
    }
    work = reinterpret_cast<unsigned long long*>(sc.p);
    unit_out = sc.p + kScratchHead;
  }
  // kernels index unit_out by absolute unit; shift the base pointer
  double2* unit_base = unit_out - (ptrdiff_t)(u0 * kNumKinds);
  // no memset: the first K2 of the valuation also writes 0 for the kinds no
  // launch group computes (zero_kinds)
  unsigned zero_kinds = ~P->payoffs & ((1u << kNumKinds) - 1);
  const int sms = device_sm_count(dev);
  const unsigned long long want = (n_units + 7) / 8;
  if (lay.engine == 3) {
    if (cnt) return fail(BP_E_INVALID_INPUT, "leaf bookkeeping runs on the class engine (constant p)");
    for (auto& g : P->groups) {
      set_units_w(g.args, u0, u1);
      const int occ = std::max(1, occupancy_exact_w(g.km));
      const int grid = (int)std::max<unsigned long long>(1, std::min<unsigned long long>(want, (unsigned long long)occ * sms));
      BP_CUDA(launch_exact_w(g.km, g.args.data(), grid, st, unit_base));
      BP_CUDA(launch_sb_reduce(unit_base, lay.units_per_sb, sb_first, sb_count, g.km, std::exchange(zero_kinds, 0u), 1.0 / P->tree.n_steps,
                               out_dev, st));
    }
  } else if (lay.engine == 2) {
    if (cnt) return fail(BP_E_INVALID_INPUT, "the threshold engine does not visit leaves (no bookkeeping)");
    ThresholdArgs a = P->th;
    {
      std::lock_guard<std::mutex> g(P->mu);
      if (!P->th_dev[dev] && !P->th_tables.empty()) {
        BP_CUDA(cudaMalloc((void**)&P->th_dev[dev], sizeof(double) * P->th_tables.size()));
        BP_CUDA(cudaMemcpyAsync(P->th_dev[dev], P->th_tables.data(), sizeof(double) * P->th_tables.size(),
                                cudaMemcpyHostToDevice, st));
      }
    }
    const size_t NL = (size_t)1 << lay.L, slot_sz = NL + NL + lay.L + 1;
    for (int slot = 0; slot < P->th_nt; ++slot) {
      a.val[slot] = P->th_dev[dev] + slot * slot_sz;
      a.pre[slot] = a.val[slot] + NL;
    }
    a.unit_first = u0;
    a.unit_end = u1;
    const int occ = std::max(1, occupancy_exact_threshold());
    const int grid = (int)std::max<unsigned long long>(1, std::min<unsigned long long>(want, (unsigned long long)occ * sms));
    BP_CUDA(launch_exact_threshold(a, grid, st, unit_base));
    BP_CUDA(launch_sb_reduce(unit_base, lay.units_per_sb, sb_first, sb_count, P->payoffs, std::exchange(zero_kinds, 0u), 1.0 / P->tree.n_steps,
                             out_dev, st));
  } else if (lay.engine == 1) {
    bool first_group = true;  // bookkeeping once per valuation, not per kind group
    for (auto& g : P->groups) {
      const bool cnt_g = cnt && first_group;
      first_group = false;
      // diagnostics: BINPATHS_K1_EMPTY=1 launches K1 with no units (its fixed cost: table setup)
      static const bool k1_empty = [] {
        const char* e = std::getenv("BINPATHS_K1_EMPTY");
        return e && std::atoi(e) != 0;
      }();
      set_units(g.args, lay.L, u0, k1_empty ? u0 : u1);
      const int occ = std::max(1, cached_occupancy_fast(lay.L, g.km, cnt_g));
      const int grid = (int)std::max<unsigned long long>(1, std::min<unsigned long long>(want, (unsigned long long)occ * sms));
      const auto tl0 = std::chrono::steady_clock::now();
      BP_CUDA(launch_exact_fast(lay.L, g.km, g.args.data(), cnt_g, grid, st, unit_base, hist_dev, g.dargs[dev], work));
      const auto tl1 = std::chrono::steady_clock::now();
      if (trace_on())
        std::fprintf(stderr, "[bp trace] K1 launch %.1f us (%zu B of arguments)\n",
                     std::chrono::duration<double, std::micro>(tl1 - tl0).count(), g.args.size());
      BP_CUDA(launch_sb_reduce(unit_base, lay.units_per_sb, sb_first, sb_count, g.km, std::exchange(zero_kinds, 0u), 1.0 / P->tree.n_steps,
                               out_dev, st, work));
    }
  } else {
    GenericArgs g = P->gen;
    g.unit_first = u0;
    g.unit_end = u1;
    const int occ = std::max(1, occupancy_exact_generic(cnt));
    const int grid = (int)std::max<unsigned long long>(1, std::min<unsigned long long>(want, (unsigned long long)occ * sms));
    BP_CUDA(launch_exact_generic(g, cnt, grid, st, unit_base, hist_dev));
    BP_CUDA(launch_sb_reduce(unit_base, lay.units_per_sb, sb_first, sb_count, P->payoffs, std::exchange(zero_kinds, 0u), 1.0, out_dev, st));
  }
  return BP_OK;
}

// Attach every class-engine group's device argument image on dev: the
// process cache, else an image the plan owns (stream-ordered allocation on
// st).  Outside any stream capture.
static int plan_attach_images(bp_exact_plan* P, int dev, cudaStream_t st) {
  if (P->lay.engine != 1) return BP_OK;
  for (auto& g : P->groups) {
    if (g.dargs[dev]) continue;
    void* p = cached_arg_image(dev, g.key, g.args);
    if (!p) {
      BP_CUDA(cudaMallocAsync(&p, g.args.size(), st));
      BP_CUDA(cudaMemcpyAsync(p, g.args.data(), g.args.size(), cudaMemcpyHostToDevice, st));
      g.dargs_owned[dev] = true;
    }
    g.dargs[dev] = p;
  }
  return BP_OK;
}

static bool plan_images_cached(const bp_exact_plan* P, int dev) {
  for (auto& g : P->groups)
    if (!g.dargs[dev] || g.dargs_owned[dev]) return false;
  return true;
}

// free the plan's own images, stream-ordered on st for device `dev_st` (the
// current device), after a device sync for the others
static void plan_release_images(bp_exact_plan* P, cudaStream_t st) {
  int cur = 0;
  cudaGetDevice(&cur);
  for (auto& g : P->groups)
    for (int d = 0; d < 64; ++d)
      if (g.dargs_owned[d] && g.dargs[d]) {
        cudaSetDevice(d);
        cudaFreeAsync(g.dargs[d], d == cur ? st : 0);
        g.dargs[d] = nullptr;
        g.dargs_owned[d] = false;
      }
  cudaSetDevice(cur);
}

static void plan_release_scratch(bp_exact_plan* P, cudaStream_t st) {
  for (int d = 0; d < 64; ++d)
    if (P->th_dev[d]) {
      int cur = 0;
      cudaGetDevice(&cur);
      cudaSetDevice(d);
      cudaDeviceSynchronize();
      cudaFree(P->th_dev[d]);
      cudaSetDevice(cur);
      P->th_dev[d] = nullptr;
    }
  for (int d = 0; d < 64; ++d)
    if (P->scratch[d].p) {
      int cur = 0;
      cudaGetDevice(&cur);
      cudaSetDevice(d);
      cudaFreeAsync(P->scratch[d].p, d == cur ? st : 0);
      cudaSetDevice(cur);
      P->scratch[d].p = nullptr;
      P->scratch[d].bytes = 0;
    }
}

static int enqueue_superblocks(const bp_tree* t, uint32_t payoffs, uint32_t flags, int dev, int sb_first,
                               int sb_count, double* out_dev, unsigned long long* hist_dev, cudaStream_t st) {
  keep_pool(dev);
  bp_exact_plan P;
  int rc = plan_build(t, payoffs, flags, &P);
  if (rc) return rc;
  rc = plan_enqueue(&P, dev, sb_first, sb_count, out_dev, hist_dev, st);
  plan_release_images(&P, st);  // stream-ordered: after the kernels
  if (P.scratch[dev].p) cudaFreeAsync(P.scratch[dev].p, st);  // stream-ordered: after the kernels
  P.scratch[dev].p = nullptr;
  if (P.th_dev[dev]) {  // K8 tables: the synchronous path frees them after the stream drains
    cudaStreamSynchronize(st);
    cudaFree(P.th_dev[dev]);
    P.th_dev[dev] = nullptr;
  }
  return rc;
}

extern "C" int bp_exact_plan_create(const bp_tree* tree, uint32_t payoffs, uint32_t flags, bp_exact_plan** out) {
  int rc = validate_tree(tree, 62, true);
  if (rc) return rc;
  if ((rc = kinds_ok(payoffs))) return rc;
  if (!out) return fail(BP_E_INVALID_INPUT, "plan pointer is NULL");
  auto* P = new bp_exact_plan();
  if ((rc = plan_build(tree, payoffs, flags, P))) {
    delete P;
    return rc;
  }
  *out = P;
  return BP_OK;
}

extern "C" int bp_exact_plan_layout(const bp_exact_plan* plan, int* n_superblocks, int* engine, int* inner_bits) {
  if (!plan) return fail(BP_E_INVALID_INPUT, "plan is NULL");
  if (n_superblocks) *n_superblocks = plan->lay.n_sb;
  if (engine) *engine = plan->lay.engine;
  if (inner_bits) *inner_bits = plan->lay.L;
  return BP_OK;
}

static bool graphs_enabled();

// The class-engine enqueue of a plan as a CUDA graph: the first enqueue for a
// (device, range, output) runs the ordinary launches (which size the plan's
// scratch); the second captures them on a private stream; later ones replay
// the graph on the caller's stream -- one launch instead of K1 (12 KB of
// arguments, ~11 us of host time) + K2.  Returns false to take the ordinary
// path.
static bool plan_enqueue_graph(bp_exact_plan* P, int dev, int sb_first, int sb_count, double* out_dev,
                               cudaStream_t st) {
  if (!graphs_enabled() || P->lay.engine != 1) return false;
  double2* scratch;
  {
    std::lock_guard<std::mutex> g(P->mu);
    scratch = P->scratch[dev].p;
    const size_t need = scratch_need((unsigned long long)sb_count * P->lay.units_per_sb);
    if (!scratch || P->scratch[dev].bytes < need) return false;  // not sized yet: ordinary path first
    const bp_exact_plan::Graph key{dev, sb_first, sb_count, out_dev, scratch, nullptr};
    for (auto it = P->graphs.begin(); it != P->graphs.end(); ++it)
      if (it->same(key)) {
        P->graphs.splice(P->graphs.begin(), P->graphs, it);  // most recently used first
        return cudaGraphLaunch(it->exec, st) == cudaSuccess;
      }
    if (!P->last_miss.same(key)) {  // first sighting: ordinary launches, capture on a repeat
      P->last_miss = key;
      return false;
    }
  }
  for (auto& g : P->groups) cached_occupancy_fast(P->lay.L, g.km, false);  // no queries inside the capture
  if (plan_attach_images(P, dev, st) != BP_OK) return false;  // uploads happen outside the capture
  cudaStream_t cap;
  if (cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking) != cudaSuccess) return false;
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  bool ok = cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal) == cudaSuccess;
  if (ok) {
    const int rc = plan_enqueue(P, dev, sb_first, sb_count, out_dev, nullptr, cap);
    ok = cudaStreamEndCapture(cap, &graph) == cudaSuccess && rc == BP_OK && graph &&
         cudaGraphInstantiate(&exec, graph, 0) == cudaSuccess;
  }
  if (graph) cudaGraphDestroy(graph);
  cudaStreamDestroy(cap);
  if (!ok) {
    cudaGetLastError();
    return false;
  }
  {
    std::lock_guard<std::mutex> g(P->mu);
    P->graphs.push_front(bp_exact_plan::Graph{dev, sb_first, sb_count, out_dev, scratch, exec});
    if (P->graphs.size() > bp_exact_plan::kMaxPlanGraphs) {
      cudaGraphExecDestroy(P->graphs.back().exec);
      P->graphs.pop_back();
    }
  }
  return cudaGraphLaunch(exec, st) == cudaSuccess;
}

extern "C" int bp_exact_plan_enqueue(bp_exact_plan* plan, int device, int sb_first, int sb_count, double* out_dev,
                                     uint64_t* hist_dev, void* stream) {
  if (!plan) return fail(BP_E_INVALID_INPUT, "plan is NULL");
  if (device < 0 || device >= bp_device_count()) return fail(BP_E_NO_DEVICE, "no CUDA device " + std::to_string(device));
  BP_CUDA(cudaSetDevice(device));
  keep_pool(device);
  const bool cnt = (plan->flags & BP_FLAG_COUNT) != 0 || hist_dev;
  if (!cnt && sb_first >= 0 && sb_count >= 1 && sb_first + sb_count <= plan->lay.n_sb &&
      plan_enqueue_graph(plan, device, sb_first, sb_count, out_dev, static_cast<cudaStream_t>(stream)))
    return BP_OK;
  return plan_enqueue(plan, device, sb_first, sb_count, out_dev, reinterpret_cast<unsigned long long*>(hist_dev),
                      static_cast<cudaStream_t>(stream));
}

extern "C" void bp_exact_plan_destroy(bp_exact_plan* plan) {
  if (!plan) return;
  for (auto& g : plan->graphs) cudaGraphExecDestroy(g.exec);
  plan_release_scratch(plan, 0);
  plan_release_images(plan, 0);
  delete plan;
}

extern "C" int bp_exact_layout(const bp_tree* tree, uint32_t payoffs, uint32_t flags, int* n_superblocks,
                               int* engine, int* inner_bits) {
  int rc = validate_tree(tree, 62, true);
  if (rc) return rc;
  if ((rc = kinds_ok(payoffs))) return rc;
  const Layout lay = choose_layout(tree, payoffs, flags, nullptr);
  if (n_superblocks) *n_superblocks = lay.n_sb;
  if (engine) *engine = lay.engine;
  if (inner_bits) *inner_bits = lay.L;
  return BP_OK;
}

extern "C" int bp_exact_superblocks(const bp_tree* tree, uint32_t payoffs, uint32_t flags, int device, int sb_first,
                                    int sb_count, double* out_dev, uint64_t* hist_dev, void* stream) {
  int rc = validate_tree(tree, 62, true);
  if (rc) return rc;
  if ((rc = kinds_ok(payoffs))) return rc;
  if (device < 0 || device >= bp_device_count()) return fail(BP_E_NO_DEVICE, "no CUDA device " + std::to_string(device));
  BP_CUDA(cudaSetDevice(device));
  return enqueue_superblocks(tree, payoffs, flags, device, sb_first, sb_count, out_dev,
                             reinterpret_cast<unsigned long long*>(hist_dev), static_cast<cudaStream_t>(stream));
}

extern "C" int bp_combine_superblocks(const double* partials, int n_sb, uint32_t payoffs, double* values) {
  if (!partials || !values || n_sb < 1) return fail(BP_E_INVALID_INPUT, "bad combine arguments");
  for (int k = 0; k < BP_N_PAYOFFS; ++k) {
    double s = 0.0, c = 0.0;
    if ((payoffs >> k) & 1)
      for (int b = 0; b < n_sb; ++b) comp_merge(s, c, partials[(b * BP_N_PAYOFFS + k) * 2], partials[(b * BP_N_PAYOFFS + k) * 2 + 1]);
    values[k] = s + c;
  }
  return BP_OK;
}

// one device's share of a synchronous valuation
struct DeviceJob {
  int device, sb_first, sb_count;
  std::vector<double> partials;       // sb_count * 6 * 2
  std::vector<unsigned long long> hist;  // 66
  float ms = 0.f;
  int rc = BP_OK;
  std::string err;
};

// Per-device resources kept across calls (stream, events, result buffers,
// pinned staging) so a synchronous valuation costs launches + one copy, not
// stream/event creation and allocations.  One call per device at a time.
struct DevCtx {
  std::mutex mu;
  bool ready = false;
  cudaStream_t st = nullptr;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  double* out_dev = nullptr;               // kMaxSB * 6 * 2
  unsigned long long* hist_dev = nullptr;  // 66
  double* out_host = nullptr;              // pinned
  unsigned long long* hist_host = nullptr; // pinned
  double2* scratch = nullptr;              // unit partials, grown on demand, kept
  size_t scratch_bytes = 0;
  // CUDA graphs of repeated synchronous valuations (class engine): key =
  // everything the captured launches depend on, most recent first
  struct Graph {
    std::vector<unsigned char> key;
    cudaGraphExec_t exec = nullptr;
  };
  std::list<Graph> graphs;
  void drop_graphs() {
    for (auto& g : graphs)
      if (g.exec) cudaGraphExecDestroy(g.exec);
    graphs.clear();
  }
};
static DevCtx g_ctx[64];

static cudaError_t ctx_init(DevCtx& c, int dev) {
  if (c.ready) return cudaSuccess;
  cudaError_t e;
  if ((e = cudaSetDevice(dev)) != cudaSuccess) return e;
  if ((e = cudaStreamCreateWithFlags(&c.st, cudaStreamNonBlocking)) != cudaSuccess) return e;
  if ((e = cudaEventCreate(&c.e0)) != cudaSuccess) return e;
  if ((e = cudaEventCreate(&c.e1)) != cudaSuccess) return e;
  if ((e = cudaMalloc((void**)&c.out_dev, sizeof(double) * kMaxSB * BP_N_PAYOFFS * 2)) != cudaSuccess) return e;
  if ((e = cudaMalloc((void**)&c.hist_dev, sizeof(unsigned long long) * 66)) != cudaSuccess) return e;
  if ((e = cudaMallocHost((void**)&c.out_host, sizeof(double) * kMaxSB * BP_N_PAYOFFS * 2)) != cudaSuccess) return e;
  if ((e = cudaMallocHost((void**)&c.hist_host, sizeof(unsigned long long) * 66)) != cudaSuccess) return e;
  c.ready = true;
  return cudaSuccess;
}

static bool graphs_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("BINPATHS_GRAPH");
    return !e || std::atoi(e) != 0;
  }();
  return on;
}

// K2 of a captured valuation writes the super-block partials straight into
// the context's pinned host buffer (device-visible under unified addressing:
// 64 x 12 posted 8-byte stores over PCIe), so the graph has no copy node
// (BINPATHS_MAPPED_OUT=0: K2 -> device buffer -> D2H copy node)
static bool mapped_out() {
  static const bool on = [] {
    const char* e = std::getenv("BINPATHS_MAPPED_OUT");
    return !e || std::atoi(e) != 0;
  }();
  return on;
}

// BINPATHS_GRAPH_EVENTS=1: the timing events are event-record nodes of the
// graph itself (no host-side record before the launch); default: recorded by
// the host around the launch
static bool graph_events() {
  static const bool on = [] {
    const char* e = std::getenv("BINPATHS_GRAPH_EVENTS");
    return e && std::atoi(e) != 0;
  }();
  return on;
}

static bool launch_graph(DevCtx& c, cudaGraphExec_t exec) {
  if (graph_events()) return cudaGraphLaunch(exec, c.st) == cudaSuccess;
  cudaEventRecord(c.e0, c.st);
  const bool ok = cudaGraphLaunch(exec, c.st) == cudaSuccess;
  cudaEventRecord(c.e1, c.st);
  return ok;
}

// Synchronous class-engine valuation as ONE graph launch: K1 (one per kind
// group), K2 and the partials' D2H copy.  The graph is captured on
// the first call for a given (argument blocks, layout, super-block range,
// scratch); a repeated valuation -- the same contract, e.g. a revaluation loop
// or the bench's e2e -- replays it (~5 us of host work instead of ~20 us of
// launches with 12 KB of kernel arguments).  Returns false to take the
// ordinary launch path (other engines, bookkeeping, or any capture failure).
// Key of a captured class-engine valuation: everything its launches depend
// on.  The K1 argument blocks are a function of the layout, the lattice
// (N, u, d, p, e^{-qT}) and the contract (S0, K), so those scalars stand for
// the 20 KB blocks; a repeated valuation finds its graph without building them.
static void graph_key(std::vector<unsigned char>& key, const Layout& lay, const bp_tree* t, uint32_t payoffs,
                      uint32_t flags, const DeviceJob* job, const double2* scratch) {
  key.clear();
  auto put = [&key](const void* p, size_t n) {
    const auto* b = static_cast<const unsigned char*>(p);
    key.insert(key.end(), b, b + n);
  };
  const double sc[6] = {t->S0, t->K, t->u, t->d, t->up_probs[0], t->disc};
  put(&lay, sizeof(lay));
  put(&payoffs, sizeof(payoffs));
  put(&flags, sizeof(flags));
  put(&job->sb_first, sizeof(int));
  put(&job->sb_count, sizeof(int));
  put(&scratch, sizeof(scratch));
  put(&t->n_steps, sizeof(t->n_steps));
  put(sc, sizeof(sc));
}

static bool try_graph_job(DevCtx& c, bp_exact_plan& P, DeviceJob* job, uint32_t flags, bool cnt) {
  if (!graphs_enabled() || cnt || P.lay.engine != 1) return false;
  const int dev = job->device;
  const unsigned long long n_units = (unsigned long long)job->sb_count * P.lay.units_per_sb;
  const size_t need = scratch_need(n_units);
  if (c.scratch_bytes < need) {  // size the scratch outside any capture; graphs on the old buffer go
    c.drop_graphs();
    if (c.scratch) cudaFreeAsync(c.scratch, c.st);
    c.scratch = nullptr;
    c.scratch_bytes = 0;
    if (scratch_alloc(&c.scratch, need, c.st) != cudaSuccess) return false;
    c.scratch_bytes = need;
  }
  for (auto& g : P.groups) cached_occupancy_fast(P.lay.L, g.km, false);  // no queries inside the capture
  // argument images from the process cache (they outlive this call's plan)
  if (plan_attach_images(&P, dev, c.st) != BP_OK || !plan_images_cached(&P, dev)) return false;
  std::vector<unsigned char> key;
  graph_key(key, P.lay, &P.tree, P.payoffs, flags, job, c.scratch);
  const size_t np = (size_t)job->sb_count * BP_N_PAYOFFS * 2;
  for (auto it = c.graphs.begin(); it != c.graphs.end(); ++it)
    if (it->key == key) {
      c.graphs.splice(c.graphs.begin(), c.graphs, it);
      return launch_graph(c, it->exec);
    }
  cudaGraph_t graph = nullptr;
  if (cudaStreamBeginCapture(c.st, cudaStreamCaptureModeThreadLocal) != cudaSuccess) return false;
  P.scratch[dev].p = c.scratch;
  P.scratch[dev].bytes = c.scratch_bytes;
  if (graph_events()) cudaEventRecordWithFlags(c.e0, c.st, cudaEventRecordExternal);
  int rc = plan_enqueue(&P, dev, job->sb_first, job->sb_count, mapped_out() ? c.out_host : c.out_dev, nullptr, c.st);
  P.scratch[dev].p = nullptr;
  P.scratch[dev].bytes = 0;
  if (!mapped_out()) cudaMemcpyAsync(c.out_host, c.out_dev, sizeof(double) * np, cudaMemcpyDeviceToHost, c.st);
  if (graph_events()) cudaEventRecordWithFlags(c.e1, c.st, cudaEventRecordExternal);
  const cudaError_t ec = cudaStreamEndCapture(c.st, &graph);
  cudaGraphExec_t exec = nullptr;
  if (rc || ec != cudaSuccess || !graph || cudaGraphInstantiate(&exec, graph, 0) != cudaSuccess) {
    if (graph) cudaGraphDestroy(graph);
    cudaGetLastError();  // clear a capture error; the caller takes the ordinary path
    return false;
  }
  cudaGraphDestroy(graph);
  c.graphs.push_front(DevCtx::Graph{std::move(key), exec});
  if (c.graphs.size() > 8) {
    cudaGraphExecDestroy(c.graphs.back().exec);
    c.graphs.pop_back();
  }
  return launch_graph(c, exec);
}

static void run_device_job(const bp_tree* t, uint32_t payoffs, uint32_t flags, DeviceJob* job) {
  auto cuda_fail = [&](cudaError_t e, const char* what) {
    job->rc = BP_E_CUDA;
    job->err = std::string("CUDA error ") + cudaGetErrorString(e) + " (" + what + ")";
  };
  if (job->device < 0 || job->device >= 64) return cuda_fail(cudaErrorInvalidDevice, "device index");
  DevCtx& c = g_ctx[job->device];
  std::lock_guard<std::mutex> lock(c.mu);
  cudaError_t e = cudaSetDevice(job->device);
  if (e != cudaSuccess) return cuda_fail(e, "cudaSetDevice");
  if ((e = ctx_init(c, job->device)) != cudaSuccess) return cuda_fail(e, "device context");
  const bool cnt = (flags & BP_FLAG_COUNT) != 0;
  const size_t np = (size_t)job->sb_count * BP_N_PAYOFFS * 2;
  job->partials.assign(np, 0.0);
  job->hist.assign(66, 0ull);
  if (cnt) cudaMemsetAsync(c.hist_dev, 0, sizeof(unsigned long long) * 66, c.st);
  keep_pool(job->device);
  // host preparation (tables) happens before the timed window
  const bool trace = trace_on();
  using clk = std::chrono::steady_clock;
  const auto t0 = clk::now();
  // a repeated class-engine valuation: its captured graph, found by key
  // before any plan is built
  if (graphs_enabled() && !cnt) {
    const Layout lay = choose_layout(t, payoffs, flags, nullptr);
    if (lay.engine == 1) {
      std::vector<unsigned char> key;
      graph_key(key, lay, t, payoffs, flags, job, c.scratch);
      for (auto it = c.graphs.begin(); it != c.graphs.end(); ++it)
        if (it->key == key) {
          c.graphs.splice(c.graphs.begin(), c.graphs, it);
          if (!launch_graph(c, it->exec)) break;
          const auto t1g = clk::now();
          if ((e = cudaStreamSynchronize(c.st)) != cudaSuccess) return cuda_fail(e, "valuation (graph)");
          if (trace)
            std::fprintf(stderr, "[bp trace] dev %d: graph key + launch %.1f us, wait %.1f us\n", job->device,
                         std::chrono::duration<double, std::micro>(t1g - t0).count(),
                         std::chrono::duration<double, std::micro>(clk::now() - t1g).count());
          std::memcpy(job->partials.data(), c.out_host, sizeof(double) * np);
          cudaEventElapsedTime(&job->ms, c.e0, c.e1);
          return;
        }
    }
  }
  bp_exact_plan P;
  int rc = plan_build(t, payoffs, flags, &P);
  const auto t1 = clk::now();
  if (!rc && P.lay.engine == 2 && !P.th_tables.empty()) {
    // K8 tables: upload before the timed window as well
    if ((e = cudaMalloc((void**)&P.th_dev[job->device], sizeof(double) * P.th_tables.size())) == cudaSuccess)
      e = cudaMemcpyAsync(P.th_dev[job->device], P.th_tables.data(), sizeof(double) * P.th_tables.size(),
                          cudaMemcpyHostToDevice, c.st);
    if (e != cudaSuccess) return cuda_fail(e, "threshold tables");
  }
  if (!rc && try_graph_job(c, P, job, flags, cnt)) {  // class engine, repeated valuation: one graph launch
    const auto t2 = clk::now();
    if ((e = cudaStreamSynchronize(c.st)) != cudaSuccess) return cuda_fail(e, "valuation (graph)");
    if (trace) {
      float gms = 0.f;
      cudaEventElapsedTime(&gms, c.e0, c.e1);
      std::fprintf(stderr, "[bp trace] dev %d: plan %.1f us, graph key + launch %.1f us, wait %.1f us (device %.1f us)\n",
                   job->device, std::chrono::duration<double, std::micro>(t1 - t0).count(),
                   std::chrono::duration<double, std::micro>(t2 - t1).count(),
                   std::chrono::duration<double, std::micro>(clk::now() - t2).count(), gms * 1e3);
    }
    std::memcpy(job->partials.data(), c.out_host, sizeof(double) * np);
    cudaEventElapsedTime(&job->ms, c.e0, c.e1);
    return;
  }
  cudaEventRecord(c.e0, c.st);
  P.scratch[job->device].p = c.scratch;  // the context's buffer (plan_enqueue grows it if needed)
  P.scratch[job->device].bytes = c.scratch_bytes;
  if (!rc) rc = plan_enqueue(&P, job->device, job->sb_first, job->sb_count, c.out_dev, cnt ? c.hist_dev : nullptr, c.st);
  c.scratch = P.scratch[job->device].p;
  c.scratch_bytes = P.scratch[job->device].bytes;
  P.scratch[job->device].p = nullptr;
  P.scratch[job->device].bytes = 0;
  if (rc) {
    job->rc = rc;
    job->err = g_err;
    cudaStreamSynchronize(c.st);
    plan_release_scratch(&P, c.st);
    plan_release_images(&P, c.st);
    return;
  }
  cudaEventRecord(c.e1, c.st);
  cudaMemcpyAsync(c.out_host, c.out_dev, sizeof(double) * np, cudaMemcpyDeviceToHost, c.st);
  if (cnt) cudaMemcpyAsync(c.hist_host, c.hist_dev, sizeof(unsigned long long) * 66, cudaMemcpyDeviceToHost, c.st);
  const auto t2 = clk::now();
  if ((e = cudaStreamSynchronize(c.st)) != cudaSuccess) return cuda_fail(e, "valuation");
  if (trace) {
    const auto t3 = clk::now();
    auto us = [](clk::duration d) { return std::chrono::duration<double, std::micro>(d).count(); };
    float kms = 0.f;
    cudaEventElapsedTime(&kms, c.e0, c.e1);
    std::fprintf(stderr, "[bp trace] dev %d: plan %.1f us, enqueue %.1f us, sync %.1f us, device %.1f us\n",
                 job->device, us(t1 - t0), us(t2 - t1), us(t3 - t2), 1e3 * kms);
  }
  std::memcpy(job->partials.data(), c.out_host, sizeof(double) * np);
  if (cnt) std::memcpy(job->hist.data(), c.hist_host, sizeof(unsigned long long) * 66);
  cudaEventElapsedTime(&job->ms, c.e0, c.e1);
  plan_release_scratch(&P, c.st);
  plan_release_images(&P, c.st);
}

extern "C" int bp_exact(const bp_tree* tree, uint32_t payoffs, uint32_t flags, int n_dev, const int* devices,
                        bp_exact_result* out) {
  const auto tb0 = std::chrono::steady_clock::now();
  int rc = validate_tree(tree, 62, true);
  if (rc) return rc;
  if ((rc = kinds_ok(payoffs))) return rc;
  if (!out) return fail(BP_E_INVALID_INPUT, "result pointer is NULL");
  const int ndev_avail = bp_device_count();
  if (ndev_avail < 1) return fail(BP_E_NO_DEVICE, "no CUDA device is visible");
  std::vector<int> devs;
  if (n_dev < 1 || !devices)
    devs.push_back(0);
  else
    devs.assign(devices, devices + n_dev);
  for (int d : devs)
    if (d < 0 || d >= ndev_avail) return fail(BP_E_NO_DEVICE, "no CUDA device " + std::to_string(d));
  const Layout lay = choose_layout(tree, payoffs, flags, nullptr);
  const int G = std::min<int>((int)devs.size(), lay.n_sb);
  std::vector<DeviceJob> jobs(G);
  int first = 0;
  for (int g = 0; g < G; ++g) {
    const int cnt = lay.n_sb / G + (g < lay.n_sb % G ? 1 : 0);
    jobs[g].device = devs[g];
    jobs[g].sb_first = first;
    jobs[g].sb_count = cnt;
    first += cnt;
  }
  const auto tb1 = std::chrono::steady_clock::now();
  if (G == 1) {
    run_device_job(tree, payoffs, flags, &jobs[0]);
    if (trace_on())
      std::fprintf(stderr, "[bp trace] bp_exact: validate + layout %.1f us, device job %.1f us\n",
                   std::chrono::duration<double, std::micro>(tb1 - tb0).count(),
                   std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - tb1).count());
  } else {
    std::vector<std::thread> th;
    for (int g = 0; g < G; ++g) th.emplace_back(run_device_job, tree, payoffs, flags, &jobs[g]);
    for (auto& x : th) x.join();
  }
  std::vector<double> all;
  std::memset(out, 0, sizeof(*out));
  float ms = 0.f;
  for (auto& j : jobs) {
    if (j.rc) return fail(j.rc, j.err);
    all.insert(all.end(), j.partials.begin(), j.partials.end());
    ms = std::max(ms, j.ms);
    for (int i = 0; i < 64; ++i) out->hist[i] += j.hist[i];
    out->leaves += j.hist[64];
    out->code_sum += j.hist[65];
  }
  bp_combine_superblocks(all.data(), lay.n_sb, payoffs, out->value);
  if (!(flags & BP_FLAG_COUNT)) out->leaves = 1ull << tree->n_steps;
  out->kernel_ms = ms;
  out->engine = lay.engine;  // 0 path walk, 1 explicit leaf tests, 2 threshold search
  out->inner_bits = lay.L;
  out->n_superblocks = lay.n_sb;
  out->n_devices = G;
  return BP_OK;
}

// ---------------------------------------------------------------------------
extern "C" void bp_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) {
  philox4x32_10(ctr[0], ctr[1], ctr[2], ctr[3], key[0], key[1], out);
}

extern "C" int bp_fp64_peak(int device, double* dfma_per_s, double* sm_clock_mhz) {
  if (device < 0 || device >= bp_device_count()) return fail(BP_E_NO_DEVICE, "no CUDA device " + std::to_string(device));
  BP_CUDA(cudaSetDevice(device));
  const int sms = device_sm_count(device);
  const int grid = sms * 8;
  double* buf = nullptr;
  unsigned long long* clk = nullptr;
  BP_CUDA(cudaMalloc((void**)&buf, sizeof(double) * grid * 256));
  BP_CUDA(cudaMalloc((void**)&clk, sizeof(unsigned long long) * 2 * grid));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  BP_CUDA(launch_dfma_peak(buf, grid, 20, 0));
  const int iters = 2000;
  cudaEventRecord(e0, 0);
  BP_CUDA(launch_dfma_peak(buf, grid, iters, 0, clk));
  cudaEventRecord(e1, 0);
  BP_CUDA(cudaEventSynchronize(e1));
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  std::vector<unsigned long long> h(2 * (size_t)grid);
  BP_CUDA(cudaMemcpy(h.data(), clk, sizeof(unsigned long long) * h.size(), cudaMemcpyDeviceToHost));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(buf);
  cudaFree(clk);
  const double ops = (double)grid * 256 * iters * 16 * 8;
  if (dfma_per_s) *dfma_per_s = ops / (ms * 1e-3);
  if (sm_clock_mhz) {
    // the clock K7 ran at: median over CTAs of SM cycles / globaltimer ns
    std::vector<double> mhz;
    for (int b = 0; b < grid; ++b)
      if (h[2 * b + 1] > 0) mhz.push_back(1e3 * (double)h[2 * b] / (double)h[2 * b + 1]);
    std::sort(mhz.begin(), mhz.end());
    *sm_clock_mhz = mhz.empty() ? 0.0 : mhz[mhz.size() / 2];
  }
  return BP_OK;
}

// ---------------------------------------------------------------------------
// Monte Carlo (mc.py:92-100,135-159,197-213,287-331)
static int single_kind(uint32_t payoff, unsigned* bit) {
  if (payoff == 0 || (payoff & (payoff - 1)) || (payoff >> BP_N_PAYOFFS))
    return fail(BP_E_INVALID_INPUT, "Monte Carlo takes exactly one payoff bit");
  *bit = (unsigned)__builtin_ctz(payoff);
  return BP_OK;
}

static void fill_mc_args(const bp_tree* t, unsigned kind, int r, uint64_t seed, uint32_t rep0, McArgs& a) {
  std::memset(&a, 0, sizeof(a));
  a.S0 = t->S0;
  a.K = t->K;
  a.u = t->u;
  a.d = t->d;
  a.invN = 1.0 / t->n_steps;
  a.N = t->n_steps;
  a.r = r;
  a.kind = kind;
  a.key0 = (uint32_t)(seed & 0xffffffffull);
  a.key1 = (uint32_t)(seed >> 32);
  philox_round_keys(a.key0, a.key1, a.rk);
  a.rep0 = rep0;
  for (int i = 0; i < t->n_steps; ++i) {
    const double p = t->up_probs[i];
    uint32_t thr = 0;
    if (p >= 1.0) {
      thr = 0xffffffffu;
      a.always[i / 32] |= 1u << (i % 32);
    } else if (p > 0.0) {
      thr = (uint32_t)std::floor(p * 4294967296.0);
    }
    a.thr[i] = thr;
  }
  // the sampler's bit planes: suffix step w = i - r sits at bit w % 32 of group w / 32;
  // T_l = threshold bit 31 - l (l < kMcLevels), up set = XOR_l (U_l & (T_{l-1} ^ T_l)) with
  // T_{-1} = T_{kMcLevels} = 0 (bp_mc_kernels.cu, draw_bits)
  for (int i = r; i < t->n_steps; ++i) {
    const int w = i - r, g = w >> 5;
    const uint32_t bit = 1u << (w & 31);
    if ((a.always[i / 32] >> (i % 32)) & 1u) {
      a.bits0[g] |= bit;
      continue;
    }
    a.open[g] |= bit;
    auto T = [&](int l) -> uint32_t { return l < 0 || l >= kMcLevels ? 0u : (a.thr[i] >> (31 - l)) & 1u; };
    if (T(0)) a.bits0[g] |= bit;
    for (int l = 0; l < kMcLevels; ++l)
      if (T(l) ^ T(l + 1)) a.flip[g][l] |= bit;
  }
}

template <typename T>
struct DevBuf {
  T* p = nullptr;
  cudaStream_t st = 0;
  ~DevBuf() {
    if (p) cudaFreeAsync(p, st);
  }
};

// Stratified MC over draw ranges [first[m], end[m]) of every stratum (first
// == nullptr: [0, end[m])).  Work items are chunks of mc_chunk() draws
// starting at first[m], so a range starting at a multiple of the chunk has
// exactly the items (and per-item statistics) of the full-range run.
static int mc_strata_ranges(const bp_tree* tree, uint32_t payoff, int r, const uint64_t* first, const uint64_t* draws,
                            uint64_t seed, uint32_t rep0, uint32_t n_reps, int device, double* theta, double* sse,
                            double* kernel_ms) {
  int rc = validate_tree(tree, 64);
  if (rc) return rc;
  unsigned kind;
  if ((rc = single_kind(payoff, &kind))) return rc;
  if (r < 0 || r > tree->n_steps || r > 24) return fail(BP_E_INVALID_INPUT, "prefix bits r out of range");
  if (!draws || !theta || !sse || n_reps < 1) return fail(BP_E_INVALID_INPUT, "bad Monte Carlo buffers");
  if (device < 0 || device >= bp_device_count()) return fail(BP_E_NO_DEVICE, "no CUDA device " + std::to_string(device));
  const int M = 1 << r;
  for (int m = 0; m < M; ++m) {
    if (draws[m] >= (1ull << 32)) return fail(BP_E_INVALID_INPUT, "at most 2^32 - 1 draws per stratum");
    if (first && first[m] > draws[m]) return fail(BP_E_INVALID_INPUT, "draw range with first > end");
  }
  // work items of one repetition, stratum-ascending: the host counts them per
  // stratum, the device lists them (launch_mc_items)
  const unsigned long long CH = mc_chunk();
  std::vector<unsigned long long> stratum_item0(M + 1, 0), first0(first ? M : 0);
  for (int m = 0; m < M; ++m) {
    const unsigned long long f = first ? first[m] : 0;
    if (first) first0[m] = f;
    stratum_item0[m + 1] = stratum_item0[m] + (draws[m] > f ? (draws[m] - f + CH - 1) / CH : 0);
  }
  const unsigned long long items_per_rep = stratum_item0[M];
  BP_CUDA(cudaSetDevice(device));
  keep_pool(device);
  cudaStream_t st;
  BP_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  struct StreamGuard {
    cudaStream_t s;
    ~StreamGuard() {
      cudaStreamSynchronize(s);
      cudaStreamDestroy(s);
    }
  } sg{st};
  McArgs a;
  fill_mc_args(tree, kind, r, seed, rep0, a);
  DevBuf<unsigned long long> d_draws, d_is, d_if, d_i0;
  DevBuf<double> d_items, d_theta, d_sse;
  d_draws.st = d_is.st = d_if.st = d_i0.st = d_items.st = d_theta.st = d_sse.st = st;
  const size_t ni = std::max<size_t>(1, items_per_rep);
  BP_CUDA(cudaMallocAsync((void**)&d_draws.p, sizeof(unsigned long long) * M, st));
  BP_CUDA(cudaMallocAsync((void**)&d_is.p, sizeof(unsigned long long) * ni, st));
  BP_CUDA(cudaMallocAsync((void**)&d_if.p, sizeof(unsigned long long) * ni, st));
  BP_CUDA(cudaMallocAsync((void**)&d_i0.p, sizeof(unsigned long long) * (M + 1), st));
  BP_CUDA(cudaMallocAsync((void**)&d_items.p, sizeof(double) * 3 * ni * n_reps, st));
  BP_CUDA(cudaMallocAsync((void**)&d_theta.p, sizeof(double) * (size_t)M * n_reps, st));
  BP_CUDA(cudaMallocAsync((void**)&d_sse.p, sizeof(double) * (size_t)M * n_reps, st));
  BP_CUDA(cudaMemcpyAsync(d_draws.p, draws, sizeof(unsigned long long) * M, cudaMemcpyHostToDevice, st));
  BP_CUDA(cudaMemcpyAsync(d_i0.p, stratum_item0.data(), sizeof(unsigned long long) * (M + 1),
                          cudaMemcpyHostToDevice, st));
  DevBuf<unsigned long long> d_first;
  d_first.st = st;
  if (first) {
    BP_CUDA(cudaMallocAsync((void**)&d_first.p, sizeof(unsigned long long) * M, st));
    BP_CUDA(cudaMemcpyAsync(d_first.p, first0.data(), sizeof(unsigned long long) * M, cudaMemcpyHostToDevice, st));
  }
  BP_CUDA(launch_mc_items(d_draws.p, d_first.p, d_i0.p, M, d_is.p, d_if.p, st));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0, st);
  BP_CUDA(launch_mc_strata(a, d_draws.p, d_is.p, d_if.p, items_per_rep, (int)n_reps, M, d_items.p, d_theta.p,
                           d_sse.p, d_i0.p, st));
  cudaEventRecord(e1, st);
  BP_CUDA(cudaMemcpyAsync(theta, d_theta.p, sizeof(double) * (size_t)M * n_reps, cudaMemcpyDeviceToHost, st));
  BP_CUDA(cudaMemcpyAsync(sse, d_sse.p, sizeof(double) * (size_t)M * n_reps, cudaMemcpyDeviceToHost, st));
  BP_CUDA(cudaStreamSynchronize(st));
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  if (kernel_ms) *kernel_ms = ms;
  return BP_OK;
}

extern "C" int bp_mc_strata(const bp_tree* tree, uint32_t payoff, int r, const uint64_t* draws, uint64_t seed,
                            uint32_t rep0, uint32_t n_reps, int device, double* theta, double* sse,
                            double* kernel_ms) {
  return mc_strata_ranges(tree, payoff, r, nullptr, draws, seed, rep0, n_reps, device, theta, sse, kernel_ms);
}

extern "C" int bp_mc_range(const bp_tree* tree, uint32_t payoff, int r, const uint64_t* first, const uint64_t* end,
                           uint64_t seed, uint32_t rep0, uint32_t n_reps, int device, double* mean, double* m2,
                           double* kernel_ms) {
  if (!first) return fail(BP_E_INVALID_INPUT, "bp_mc_range needs the first draw of every stratum");
  return mc_strata_ranges(tree, payoff, r, first, end, seed, rep0, n_reps, device, mean, m2, kernel_ms);
}

extern "C" int bp_mc_shared(const bp_tree* tree, uint32_t payoff, int r, uint64_t R, const double* masses,
                            uint64_t seed, uint32_t rep0, uint32_t n_reps, int device, double* inner_mean,
                            double* inner_sse, double* stratum_means, double* kernel_ms) {
  int rc = validate_tree(tree, 64);
  if (rc) return rc;
  unsigned kind;
  if ((rc = single_kind(payoff, &kind))) return rc;
  if (r < 0 || r > tree->n_steps || r > 16) return fail(BP_E_INVALID_INPUT, "prefix bits r out of range");
  if (R < 1 || R >= (1ull << 32)) return fail(BP_E_INVALID_INPUT, "R must be in [1, 2^32)");
  if (!masses || !inner_mean || !inner_sse || !stratum_means || n_reps < 1)
    return fail(BP_E_INVALID_INPUT, "bad Monte Carlo buffers");
  if (device < 0 || device >= bp_device_count()) return fail(BP_E_NO_DEVICE, "no CUDA device " + std::to_string(device));
  const int M = 1 << r;
  // prefix states (S, sum, max, min) after the r prefix steps of every stratum
  std::vector<double> pre(4 * (size_t)M);
  for (int m = 0; m < M; ++m) {
    double S = tree->S0, sum = 0.0, mx = -INFINITY, mn = INFINITY;
    for (int t = 0; t < r; ++t) {
      const int b = (m >> (r - 1 - t)) & 1;
      S *= b ? tree->u : tree->d;
      sum += S;
      mx = std::max(mx, S);
      mn = std::min(mn, S);
    }
    pre[4 * m] = S;
    pre[4 * m + 1] = sum;
    pre[4 * m + 2] = mx;
    pre[4 * m + 3] = mn;
  }
  const unsigned long long CH = mc_chunk();
  const unsigned long long items_per_rep = (R + CH - 1) / CH;
  BP_CUDA(cudaSetDevice(device));
  keep_pool(device);
  cudaStream_t st;
  BP_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  struct StreamGuard {
    cudaStream_t s;
    ~StreamGuard() {
      cudaStreamSynchronize(s);
      cudaStreamDestroy(s);
    }
  } sg{st};
  McArgs a;
  fill_mc_args(tree, kind, r, seed, rep0, a);
  DevBuf<double> d_m, d_pre, d_items, d_ws, d_im, d_is, d_sm;
  d_m.st = d_pre.st = d_items.st = d_ws.st = d_im.st = d_is.st = d_sm.st = st;
  const size_t nit = (size_t)items_per_rep * n_reps;
  BP_CUDA(cudaMallocAsync((void**)&d_m.p, sizeof(double) * M, st));
  BP_CUDA(cudaMallocAsync((void**)&d_pre.p, sizeof(double) * 4 * M, st));
  BP_CUDA(cudaMallocAsync((void**)&d_items.p, sizeof(double) * 3 * nit, st));
  BP_CUDA(cudaMallocAsync((void**)&d_ws.p, sizeof(double) * 8 * nit * M, st));
  BP_CUDA(cudaMallocAsync((void**)&d_im.p, sizeof(double) * n_reps, st));
  BP_CUDA(cudaMallocAsync((void**)&d_is.p, sizeof(double) * n_reps, st));
  BP_CUDA(cudaMallocAsync((void**)&d_sm.p, sizeof(double) * (size_t)M * n_reps, st));
  BP_CUDA(cudaMemcpyAsync(d_m.p, masses, sizeof(double) * M, cudaMemcpyHostToDevice, st));
  BP_CUDA(cudaMemcpyAsync(d_pre.p, pre.data(), sizeof(double) * 4 * M, cudaMemcpyHostToDevice, st));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0, st);
  BP_CUDA(launch_mc_shared(a, R, d_m.p, d_pre.p, M, (int)n_reps, d_items.p, d_ws.p, items_per_rep, d_im.p, d_is.p,
                           d_sm.p, st));
  cudaEventRecord(e1, st);
  BP_CUDA(cudaMemcpyAsync(inner_mean, d_im.p, sizeof(double) * n_reps, cudaMemcpyDeviceToHost, st));
  BP_CUDA(cudaMemcpyAsync(inner_sse, d_is.p, sizeof(double) * n_reps, cudaMemcpyDeviceToHost, st));
  BP_CUDA(cudaMemcpyAsync(stratum_means, d_sm.p, sizeof(double) * (size_t)M * n_reps, cudaMemcpyDeviceToHost, st));
  BP_CUDA(cudaStreamSynchronize(st));
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  if (kernel_ms) *kernel_ms = ms;
  return BP_OK;
}

// ---------------------------------------------------------------------------
// batched exact pricing (K3)
extern "C" int bp_exact_batch(const bp_tree* trees, int n_opts, uint32_t payoff, int device, double* values,
                              double* kernel_ms) {
  if (!trees || n_opts < 1 || !values) return fail(BP_E_INVALID_INPUT, "bad batch arguments");
  unsigned kind;
  int rc = single_kind(payoff, &kind);
  if (rc) return rc;
  const int N = trees[0].n_steps;
  if (N < kFastMinN || N > 40) return fail(BP_E_INVALID_INPUT, "batched pricing supports 16 <= N <= 40");
  std::vector<BatchOption> h(n_opts);
  for (int i = 0; i < n_opts; ++i) {
    const bp_tree* t = &trees[i];
    if ((rc = validate_tree(t, 62))) return rc;
    if (t->n_steps != N) return fail(BP_E_LENGTH_MISMATCH, "all trees of a batch must have the same N");
    if (!constant_p(t)) return fail(BP_E_NONCONSTANT_PROBS, "batched pricing needs a constant up probability");
    if (!(t->u > t->d)) return fail(BP_E_INVALID_INPUT, "batched pricing needs u > d");
    h[i] = BatchOption{t->S0, t->K, t->u, t->d, t->up_probs[0], t->disc};
  }
  if (device < 0 || device >= bp_device_count()) return fail(BP_E_NO_DEVICE, "no CUDA device " + std::to_string(device));
  BP_CUDA(cudaSetDevice(device));
  keep_pool(device);
  cudaStream_t st;
  BP_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  struct StreamGuard {
    cudaStream_t s;
    ~StreamGuard() {
      cudaStreamSynchronize(s);
      cudaStreamDestroy(s);
    }
  } sg{st};
  const BatchLayout blay = batch_layout(n_opts, N);
  DevBuf<BatchOption> d_o;
  DevBuf<double> d_v;
  DevBuf<double2> d_p;
  d_o.st = d_v.st = d_p.st = st;
  BP_CUDA(cudaMallocAsync((void**)&d_o.p, sizeof(BatchOption) * n_opts, st));
  BP_CUDA(cudaMallocAsync((void**)&d_v.p, sizeof(double) * n_opts, st));
  BP_CUDA(cudaMallocAsync((void**)&d_p.p, sizeof(double2) * (size_t)blay.ctas(), st));
  BP_CUDA(cudaMemcpyAsync(d_o.p, h.data(), sizeof(BatchOption) * n_opts, cudaMemcpyHostToDevice, st));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0, st);
  BP_CUDA(launch_exact_batch(d_o.p, blay, N, kind, d_v.p, d_p.p, st));
  cudaEventRecord(e1, st);
  BP_CUDA(cudaMemcpyAsync(values, d_v.p, sizeof(double) * n_opts, cudaMemcpyDeviceToHost, st));
  BP_CUDA(cudaStreamSynchronize(st));
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  if (kernel_ms) *kernel_ms = ms;
  return BP_OK;
}

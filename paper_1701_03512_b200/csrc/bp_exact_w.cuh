// Arguments of the per-leaf-weight enumeration kernel K1w (bp_exact_w_kernels.cu).
#pragma once
#include <type_traits>
#include "bp_exact.cuh"

namespace bp {

struct ExactWScalars {
  double S0, K, NK, u, d, disc;
  double E;      // sum_s w_s e_s over the inner block (floating lookback)
  double Omega;  // sum_s w_s over the inner block (1 up to rounding)
  int N, L, D, m, Dp, n_mid, q, zero;
  unsigned long long unit_first, unit_end;
};

// leaves per sorted group (one prefix-sum lookup) and per independent count
// chain inside a group (as K1's kGroup / kChain; bp_exact.cuh)
constexpr int kWGroup = 32, kWChain = 4;

template <int L>
struct __align__(16) ExactWArgs {
  double tab[2 << L];                  // per slot: inner values sorted in the compare direction
  double2 gp[2][(1 << L) / kWGroup * (kWGroup + 1)];  // per slot and group: (sum w v, sum w) of the first n
  double mid_c[kMidMax], mid_e[kMidMax], mid_mx[kMidMax], mid_mn[kMidMax], mid_w[kMidMax];
  double p[kMaxN], q[kMaxN];           // prefix steps: p_t and 1 - p_t
  ExactWScalars s;
};

}  // namespace bp

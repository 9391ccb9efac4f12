// Arguments of the threshold-search engine (K8, bp_threshold_kernels.cu).
#pragma once
#include "bp_kernels.h"

namespace bp {

struct ThresholdArgs {
  const double* val[4];   // per kind slot: class-sorted values, 2^LT
  const double* pre[4];   // per kind slot: class prefix sums, 2^LT + LT + 1
  int class_off[kMaxThreshL + 2];  // start of class c in val (c = 0..LT+1)
  double w[kMaxN + 2 + kMaxThreshL + 1];
  double e_cls[kMaxThreshL + 1], b_cls[kMaxThreshL + 1];
  double S0, K, NK, u, d;
  int N, LT, D, m, Dp, q;
  unsigned kinds;
  unsigned long long unit_first, unit_end;
};

}  // namespace bp

// Internal launch interface between the kernel translation units and the
// C ABI (bp_capi.cu).  Not part of the public header.
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>
#include "bp_exact.cuh"

namespace bp {

bool fast_kind_mask_supported(unsigned km);
// dev_args: a device copy of the argument block's tables (CTA setup reads).
// work: the unit counter of the launch (device, 0 on entry; the K2 launched
// after it resets it)
cudaError_t launch_exact_fast(int L, unsigned km, const void* args, bool cnt, int grid, cudaStream_t st,
                              double2* unit_out, unsigned long long* hist, const void* dev_args,
                              unsigned long long* work);
int occupancy_exact_fast(int L, unsigned km, bool cnt);
size_t exact_args_size(int L);

cudaError_t launch_exact_generic(const GenericArgs& a, bool cnt, int grid, cudaStream_t st, double2* unit_out,
                                 unsigned long long* hist);
int occupancy_exact_generic(bool cnt);

// work: a K1 unit counter to reset to 0 (stream order: after that K1), or nullptr
cudaError_t launch_sb_reduce(const double2* unit_out, unsigned long long units_per_sb, int sb_first, int sb_count,
                             unsigned kinds, unsigned zero_kinds, double scale_asian, double* out, cudaStream_t st,
                             unsigned long long* work = nullptr);

// Batched exact (one option per CTA group), see bp_batch_kernels.cu
struct BatchOption {
  double S0, K, u, d, p, disc;
};
// CTA layout of a batch: options [0, n_whole) get 2^base_log2 CTAs each, the
// tail options [n_whole, n_opts) 2^tail_log2 each (the last wave's options are
// split so it is not a mostly idle wave)
struct BatchLayout {
  int n_opts, n_whole, base_log2, tail_log2;
  long long ctas() const {
    return ((long long)n_whole << base_log2) + ((long long)(n_opts - n_whole) << tail_log2);
  }
};
BatchLayout batch_layout(int n_opts, int N);
cudaError_t launch_exact_batch(const BatchOption* opts_dev, const BatchLayout& lay, int N, unsigned kind,
                               double* values_dev, double2* scratch_dev, cudaStream_t st);

// Monte Carlo, see bp_mc_kernels.cu
constexpr int kMcLevels = 8;  // threshold bits compared bit-sliced before the tie words
struct McArgs {
  double S0, K, u, d, invN;
  uint32_t thr[kMaxN];   // Bernoulli thresholds floor(p_t 2^32) (saturated)
  uint32_t always[2];    // bit t set: step t is always up (p_t >= 1)
  // bit-sliced sampler (bp_mc_kernels.cu): suffix step w = 32 g + b is bit b of group g
  uint32_t flip[2][kMcLevels];  // C_{l+1}: steps whose threshold bits 31 - l and 30 - l differ (bit -1 = 0)
  uint32_t bits0[2];            // steps that are always up, and U_0 & C_0 (threshold bit 31 set)
  uint32_t open[2];             // U_0: steps decided by the stream (valid and not forced)
  int N, r;
  unsigned kind;
  uint32_t key0, key1;
  uint32_t rk[20];  // Philox round keys of (key0, key1)
  uint32_t rep0;
};
// item lists of one repetition: stratum m's chunks of mc_chunk() draws from first[m] (nullptr: 0) to draws[m]
cudaError_t launch_mc_items(const unsigned long long* draws_dev, const unsigned long long* first_dev,
                            const unsigned long long* stratum_item0_dev, int n_strata,
                            unsigned long long* item_stratum_dev, unsigned long long* item_first_dev, cudaStream_t st);
cudaError_t launch_mc_strata(const McArgs& a, const unsigned long long* draws_dev,
                             const unsigned long long* item_stratum_dev, const unsigned long long* item_first_dev,
                             unsigned long long items_per_rep, int n_reps, int n_strata, double* item_out_dev,
                             double* theta_dev, double* sse_dev, const unsigned long long* stratum_item0_dev,
                             cudaStream_t st);
cudaError_t launch_mc_shared(const McArgs& a, unsigned long long R, const double* masses_dev, const double* pre_tab_dev,
                             int M, int n_reps, double* item_out_dev, double* warp_sums_dev,
                             unsigned long long items_per_rep, double* inner_mean_dev, double* inner_sse_dev,
                             double* stratum_means_dev, cudaStream_t st);
unsigned long long mc_chunk();

cudaError_t launch_dfma_peak(double* out, int grid, int iters, cudaStream_t st,
                             unsigned long long* clk = nullptr);

// K1w per-leaf-weight enumeration (any per-step probabilities), bp_exact_w_kernels.cu
cudaError_t launch_exact_w(unsigned km, const void* args, int grid, cudaStream_t st, double2* unit_out);
int occupancy_exact_w(unsigned km);

// K8 threshold-search engine, see bp_threshold_kernels.cu
constexpr int kMaxThreshL = 22;
struct ThresholdArgs;
cudaError_t launch_exact_threshold(const ThresholdArgs& a, int grid, cudaStream_t st, double2* unit_out);
int occupancy_exact_threshold();

// the K1 (L, kind mask) instantiations: every single kind plus the fused
// config-2 pair (Asian call + floating lookback)
#define BP_FAST_KMS(X, L)                                                      \
  X(L, (1u << kAC)) X(L, (1u << kAP)) X(L, (1u << kFL)) X(L, (1u << kFLP))     \
  X(L, (1u << kEC)) X(L, (1u << kEP)) X(L, ((1u << kAC) | (1u << kFL)))
constexpr int kFastParts = 14;  // BP_FAST_KMS x L in {8, 9}: parts of bp_exact_fast_inst.cu

}  // namespace bp

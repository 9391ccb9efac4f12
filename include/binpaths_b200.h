/*
 * binpaths_b200.h — C ABI of the B200 engine for the exact 2^N path
 * enumeration and the stratified Monte Carlo estimators of arXiv 1701.03512.
 *
 * Plain C types only (no torch, no CUDA types in signatures).  Every entry
 * point returns a status code (BP_OK == 0); on failure bp_last_error()
 * returns a thread-local message.  Status codes map one-to-one onto the
 * reference's exception classes (pkg/src/binpaths/errors.py:4-41), see
 * bp_status below.  The host mirror in paper_1701_03512_b200/_native.py
 * raises the same Python classes.
 *
 * Reference interfaces replaced (paths relative to /root/reference):
 *   bp_exact             value_exact_serial / value_exact_parallel
 *                        (pkg/src/binpaths/exact.py:103-133)
 *   bp_exact_superblocks _rank_value for a power-of-two rank
 *                        (pkg/src/binpaths/exact.py:83-100,
 *                        partition of paths.py:103-123,141-145)
 *   bp_combine_superblocks  ascending-rank reduction (exact.py:130-133)
 *   bp_exact_batch       a loop of value_exact_parallel over requests
 *                        (no batch API in the reference)
 *   bp_mc_strata         _stratum_stats over all strata of a plan
 *                        (pkg/src/binpaths/mc.py:197-213, sampler
 *                        mc.py:92-100); with r = 0 it is estimate_basic's
 *                        draw loop (mc.py:135-159)
 *   bp_mc_range          _stratum_stats over draw slices (one process per
 *                        GPU: basic MC's draws split by rank)
 *   bp_mc_shared         the draw loop of estimate_shared (mc.py:287-331)
 *   bp_philox4x32_10     counter-based generator used by bp_mc_* (stands in
 *                        for numpy Philox keyed by SeedSequence, mc.py:92-95)
 */
#ifndef BINPATHS_B200_H
#define BINPATHS_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BP_ABI_VERSION 1

/* ---- payoff kinds (bit mask) -------------------------------------------
 * The four reference kinds (payoffs.py:24-28) and the two BASELINE kinds the
 * reference reaches only through its callable extension point
 * (payoffs.py:33-34, 66-70).  All payoffs see S_1..S_N, never S_0.      */
enum bp_payoff {
    BP_EURO_CALL          = 1u << 0, /* max(S_N - K, 0)                  */
    BP_EURO_PUT           = 1u << 1, /* max(K - S_N, 0)                  */
    BP_ASIAN_PUT          = 1u << 2, /* max(K - mean(S_1..S_N), 0)       */
    BP_FIXED_LOOKBACK_PUT = 1u << 3, /* max(K - min(S_1..S_N), 0)        */
    BP_ASIAN_CALL         = 1u << 4, /* max(mean(S_1..S_N) - K, 0)       */
    BP_FLOAT_LOOKBACK     = 1u << 5  /* max(S_1..S_N) - S_N              */
};
#define BP_N_PAYOFFS 6

/* ---- status codes ------------------------------------------------------ */
enum bp_status {
    BP_OK                   = 0,
    BP_E_INVALID_INPUT      = 1, /* InvalidInput          errors.py:8  */
    BP_E_PROBABILITY        = 2, /* ProbabilityOutOfRange errors.py:12 */
    BP_E_LENGTH_MISMATCH    = 3, /* LengthMismatch        errors.py:16 */
    BP_E_WORKER_COUNT       = 4, /* InvalidWorkerCount    errors.py:20 */
    BP_E_RANK_RANGE         = 5, /* RankOutOfRange        errors.py:24 */
    BP_E_PATH_DEPENDENT     = 6, /* PathDependentPayoff   errors.py:28 */
    BP_E_NONCONSTANT_PROBS  = 7, /* NonConstantProbs      errors.py:32 */
    BP_E_INFEASIBLE_ALLOC   = 8, /* InfeasibleAllocation  errors.py:36 */
    BP_E_ENUMERATION_GUARD  = 9, /* EnumerationGuard      errors.py:40 */
    BP_E_CUDA               = 100,
    BP_E_NO_DEVICE          = 101
};

/* ---- flags ------------------------------------------------------------- */
#define BP_FLAG_COUNT       1u  /* leaf bookkeeping: per-up-count histogram */
#define BP_FLAG_GENERIC     2u  /* force the per-path walk kernel           */
#define BP_FLAG_NO_TIMING   4u  /* skip the CUDA-event timing of the launch */
#define BP_FLAG_THRESHOLD   8u  /* threshold-search engine: per node, binary
                                   search of the class-sorted inner tables;
                                   leaves are NOT visited one by one, report
                                   its rate as "effective paths/s"          */

/* One tree + contract.  Mirrors the fields the reference engine reads:
 * inputs.{S0,K,N} and params.{u,d,up_probs} (exact.py:87-99), with the
 * discount e^{-qT} precomputed (exact.py:99).                            */
typedef struct bp_tree {
    int32_t n_steps;          /* N, 1..62 (64 for bp_mc_*)                */
    int32_t reserved;
    double S0;                /* finite; bp_exact* also take S0 <= 0     *
                               * (per-path walk, as the reference reads   *
                               * S0 unchecked, exact.py:96,99); > 0 for   *
                               * bp_mc_* and bp_exact_batch               */
    double K;                 /* strike                                  */
    double u;                 /* up factor   (> 0)                       */
    double d;                 /* down factor (> 0)                       */
    double disc;              /* e^{-qT}                                 */
    const double* up_probs;   /* n_steps per-step up probabilities (host) */
} bp_tree;

/* Result of one exact valuation. */
typedef struct bp_exact_result {
    double   value[BP_N_PAYOFFS]; /* discounted value, index = bit position  */
    uint64_t leaves;              /* paths the kernels visited (== 2^N)       */
    uint64_t code_sum;            /* sum of visited path codes (mod 2^64)     */
    uint64_t hist[64];            /* BP_FLAG_COUNT: leaves per up-count h     */
    double   kernel_ms;           /* device time of the valuation (events)    */
    int32_t  engine;              /* 0 path walk, 1 leaf tests, 2 search      */
    int32_t  inner_bits;          /* L, leaves per inner block = 2^L          */
    int32_t  n_superblocks;       /* canonical partial count                  */
    int32_t  n_devices;
} bp_exact_result;

/* Exact expected value over all 2^N paths (value_exact_parallel).
 * payoffs: OR of bp_payoff bits.  devices: n_dev CUDA ordinals (n_dev >= 1);
 * contiguous ranges of the canonical super-blocks go to them, one host
 * thread per device.  The result is bitwise independent of n_dev.        */
int bp_exact(const bp_tree* tree, uint32_t payoffs, uint32_t flags,
             int n_dev, const int* devices, bp_exact_result* out);

/* Number of canonical super-blocks of a valuation (64 when 2^N is large).  */
int bp_exact_layout(const bp_tree* tree, uint32_t payoffs, uint32_t flags,
                    int* n_superblocks, int* engine, int* inner_bits);

/* Asynchronous shard step for one process per GPU: computes the partials of
 * super-blocks [sb_first, sb_first + sb_count) on `device`, enqueued on the
 * CUDA stream `stream` (a cudaStream_t; NULL = legacy default stream).
 * out_dev: DEVICE buffer of sb_count * BP_N_PAYOFFS * 2 doubles, laid out
 * [sb][payoff bit][sum, compensation].  hist_dev: DEVICE buffer of 66
 * uint64 (hist[64], leaves, code_sum) accumulated atomically, or NULL.
 * The call returns once the work is enqueued.                             */
int bp_exact_superblocks(const bp_tree* tree, uint32_t payoffs, uint32_t flags,
                         int device, int sb_first, int sb_count,
                         double* out_dev, uint64_t* hist_dev, void* stream);

/* A prepared valuation (kernel arguments and tables built once, scratch
 * reused): for repeated valuations of one tree, e.g. one step per rank in a
 * one-process-per-GPU job.  Enqueue has the semantics of
 * bp_exact_superblocks; calls on one plan and device must use one stream.
 * Replaces the per-call setup of _rank_value (exact.py:83-100).            */
typedef struct bp_exact_plan bp_exact_plan;
int bp_exact_plan_create(const bp_tree* tree, uint32_t payoffs, uint32_t flags,
                         bp_exact_plan** plan);
int bp_exact_plan_layout(const bp_exact_plan* plan, int* n_superblocks,
                         int* engine, int* inner_bits);
int bp_exact_plan_enqueue(bp_exact_plan* plan, int device, int sb_first,
                          int sb_count, double* out_dev, uint64_t* hist_dev,
                          void* stream);
void bp_exact_plan_destroy(bp_exact_plan* plan);

/* Fixed-order (ascending super-block) compensated combination of the
 * gathered partials (host memory, n_sb * BP_N_PAYOFFS * 2 doubles) into
 * the discounted values (BP_N_PAYOFFS doubles).                            */
int bp_combine_superblocks(const double* partials, int n_sb, uint32_t payoffs,
                           double* values);

/* Batched exact pricing: n_opts independent trees (constant up probability
 * each, same N), one payoff kind, one device.  values: n_opts doubles.   */
int bp_exact_batch(const bp_tree* trees, int n_opts, uint32_t payoff,
                   int device, double* values, double* kernel_ms);

/* Stratified Monte Carlo statistics.  The first r steps of every draw of
 * stratum m are the r binary digits of m (step 1 = most significant); the
 * remaining N - r steps are Bernoulli(floor(up_probs[t] 2^32) / 2^32) draws
 * from Philox4x32-10 with key = seed and counter = (word-block, draw,
 * stratum, rep); which word decides which step (32 steps per word, 8
 * threshold bits, then tie words) is laid out in csrc/bp_mc_kernels.cu's
 * header and restated step by step in oracle/bp_oracle.c (mc_suffix_bits).
 * Results depend on (seed, stratum, rep, draw index) only, never on the
 * grid, the device or the split into ranges.  For stratum m and repetition rep0 + k it writes the mean theta and
 * the sum of squared deviations sse of the draws[m] payoffs (undiscounted,
 * the theta scale of mc.py:197-213).  Strata with draws[m] == 0 report
 * (0, 0).  Outputs are [n_reps][2^r] arrays in host memory.            */
int bp_mc_strata(const bp_tree* tree, uint32_t payoff, int r,
                 const uint64_t* draws, uint64_t seed, uint32_t rep0,
                 uint32_t n_reps, int device, double* theta, double* sse,
                 double* kernel_ms);

/* Shared-sample Monte Carlo (estimate_shared, mc.py:287-331): R suffix draws
 * on the stratum-0 stream, each evaluated under all 2^r prefixes; inner =
 * sum_m masses[m] * payoff(m, draw).  Writes, per repetition, the mean and
 * sse of the inner sums and the per-stratum payoff means ([n_reps][2^r]). */
/* bp_mc_strata over draw RANGES: stratum m contributes draws
 * [first[m], end[m]) of its stream (same draws as in the full run).  It
 * writes the range's mean and sum of squared deviations (mean, m2; count =
 * end - first) per stratum and repetition.  For one process per GPU: a
 * range starting at a multiple of 4096 draws is evaluated exactly as in the
 * full run; the ranks' (count, mean, m2) are merged with Chan's formula in
 * rank order.  Replaces _stratum_stats over a slice of draws (mc.py:197-213). */
int bp_mc_range(const bp_tree* tree, uint32_t payoff, int r,
                const uint64_t* first, const uint64_t* end, uint64_t seed,
                uint32_t rep0, uint32_t n_reps, int device, double* mean,
                double* m2, double* kernel_ms);

int bp_mc_shared(const bp_tree* tree, uint32_t payoff, int r, uint64_t R,
                 const double* masses, uint64_t seed, uint32_t rep0,
                 uint32_t n_reps, int device, double* inner_mean,
                 double* inner_sse, double* stratum_means, double* kernel_ms);

/* Philox4x32-10 block function (host implementation of the device
 * generator, exported for known-answer tests).  ctr[4], key[2] -> out[4]. */
void bp_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2],
                      uint32_t out[4]);

/* Measured FP64-pipe peak (DFMA per second) of a device: a microbenchmark
 * of independent DFMA chains over every SM (K7 of SURVEY.md §2.3), and the
 * SM clock it ran at (median over CTAs of clock64 cycles per globaltimer ns),
 * so the rate can be compared with n_SM x 64 x clock.                      */
int bp_fp64_peak(int device, double* dfma_per_s, double* sm_clock_mhz);

int bp_device_count(void);
int bp_abi_version(void);
const char* bp_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* BINPATHS_B200_H */

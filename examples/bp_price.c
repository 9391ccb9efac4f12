/*
 * bp_price.c -- a plain C caller of the engine's C ABI (include/binpaths_b200.h):
 * no Python, no torch, no CUDA headers.  It prices BASELINE configs[0] (N = 20
 * Asian call, classic CRR; golden 6.029007913100635 from the reference,
 * tests/golden/exact_config1.json) and the floating lookback in one call, prints
 * the values, the leaf bookkeeping and the per-call wall time, and exercises the
 * error path (EnumerationGuard-style status for a bad tree).
 *
 *   cc -O2 -I include examples/bp_price.c -L paper_1701_03512_b200/_lib \
 *      -lbinpaths_b200 -Wl,-rpath,'$ORIGIN/../paper_1701_03512_b200/_lib' -lm
 *   ./bp_price [N]          exit 0 = ok, 1 = engine error, 2 = parity failure
 */
#define _POSIX_C_SOURCE 199309L
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <time.h>

#include "binpaths_b200.h"

static double now_s(void) {
    struct timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    return ts.tv_sec + 1e-9 * ts.tv_nsec;
}

int main(int argc, char** argv) {
    const int N = argc > 1 ? atoi(argv[1]) : 20;
    const double S0 = 100.0, K = 100.0, r = 0.05, sigma = 0.2, T = 1.0;
    const double dt = T / N, u = exp(sigma * sqrt(dt)), d = 1.0 / u;
    const double p = (exp(r * dt) - d) / (u - d);
    double* probs = malloc(sizeof(double) * N);
    for (int i = 0; i < N; ++i) probs[i] = p;
    bp_tree tree = {N, 0, S0, K, u, d, exp(-r * T), probs};

    if (bp_device_count() < 1) {
        fprintf(stderr, "no CUDA device: %s\n", bp_last_error());
        return 1;
    }
    bp_exact_result res;
    const uint32_t kinds = BP_ASIAN_CALL | BP_FLOAT_LOOKBACK;
    int rc = bp_exact(&tree, kinds, BP_FLAG_COUNT, 0, NULL, &res); /* warm-up (context, plan cache) */
    const double t0 = now_s();
    rc = rc ? rc : bp_exact(&tree, kinds, BP_FLAG_COUNT, 0, NULL, &res);
    const double wall = now_s() - t0;
    if (rc) {
        fprintf(stderr, "bp_exact failed (%d): %s\n", rc, bp_last_error());
        return 1;
    }
    printf("N=%d asian-call=%.15g float-lookback=%.15g leaves=%llu engine=%d kernel_ms=%.3f wall_ms=%.3f\n", N,
           res.value[4], res.value[5], (unsigned long long)res.leaves, res.engine, res.kernel_ms, wall * 1e3);

    /* bookkeeping: leaves per up count == C(N, h), total 2^N */
    double c = 1.0;
    for (int h = 0; h <= N; ++h) {
        if ((double)res.hist[h] != c) {
            fprintf(stderr, "hist[%d] = %llu, want %.0f\n", h, (unsigned long long)res.hist[h], c);
            return 2;
        }
        c = c * (N - h) / (h + 1);
    }
    if (res.leaves != (1ull << N)) return 2;
    if (N == 20 && fabs(res.value[4] - 6.029007913100635) > 1e-12 * 6.029007913100635) {
        fprintf(stderr, "asian-call %.17g differs from the reference golden\n", res.value[4]);
        return 2;
    }

    /* error path: a probability outside (0, 1) is ProbabilityOutOfRange */
    probs[0] = 1.5;
    rc = bp_exact(&tree, kinds, 0, 0, NULL, &res);
    printf("bad tree -> status %d (%s)\n", rc, bp_last_error());
    free(probs);
    return rc == BP_E_PROBABILITY ? 0 : 2;
}

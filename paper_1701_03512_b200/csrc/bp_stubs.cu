// Temporary: entry points whose kernels land in the next commit.
#include "../../include/binpaths_b200.h"
#include <string>
extern "C" int bp_exact_batch(const bp_tree*, int, uint32_t, int, double*, double*) { return BP_E_INVALID_INPUT; }
extern "C" int bp_mc_strata(const bp_tree*, uint32_t, int, const uint64_t*, uint64_t, uint32_t, uint32_t, int, double*, double*, double*) { return BP_E_INVALID_INPUT; }
extern "C" int bp_mc_shared(const bp_tree*, uint32_t, int, uint64_t, const double*, uint64_t, uint32_t, uint32_t, int, double*, double*, double*, double*) { return BP_E_INVALID_INPUT; }

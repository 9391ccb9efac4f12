// Temporary: the batched entry point lands with its kernel in the next commit.
#include "../../include/binpaths_b200.h"
extern "C" int bp_exact_batch(const bp_tree*, int, uint32_t, int, double*, double*) { return BP_E_INVALID_INPUT; }

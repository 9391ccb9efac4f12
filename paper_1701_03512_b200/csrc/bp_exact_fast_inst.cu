// One K1 instantiation per translation unit: build.py compiles this file
// kFastParts times with -DBP_FAST_PART=i, instantiating the i-th (L, kind
// mask) pair of BP_FAST_LS (bp_kernels.h), so the 14 fully unrolled kernels
// compile in parallel.
#include "bp_exact_fast.cuh"

namespace bp {

#define BP_INST(LL, KMV)                                                                              \
  template cudaError_t launch_fast_t<LL, KMV>(const void*, bool, int, cudaStream_t, double2*,        \
                                              unsigned long long*, const void*, unsigned long long*); \
  template int occupancy_fast_t<LL, KMV>(bool);

#if BP_FAST_PART == 0
BP_INST(8, (1u << kAC))
#elif BP_FAST_PART == 1
BP_INST(8, (1u << kAP))
#elif BP_FAST_PART == 2
BP_INST(8, (1u << kFL))
#elif BP_FAST_PART == 3
BP_INST(8, (1u << kFLP))
#elif BP_FAST_PART == 4
BP_INST(8, (1u << kEC))
#elif BP_FAST_PART == 5
BP_INST(8, (1u << kEP))
#elif BP_FAST_PART == 6
BP_INST(8, ((1u << kAC) | (1u << kFL)))
#elif BP_FAST_PART == 7
BP_INST(9, (1u << kAC))
#elif BP_FAST_PART == 8
BP_INST(9, (1u << kAP))
#elif BP_FAST_PART == 9
BP_INST(9, (1u << kFL))
#elif BP_FAST_PART == 10
BP_INST(9, (1u << kFLP))
#elif BP_FAST_PART == 11
BP_INST(9, (1u << kEC))
#elif BP_FAST_PART == 12
BP_INST(9, (1u << kEP))
#elif BP_FAST_PART == 13
BP_INST(9, ((1u << kAC) | (1u << kFL)))
#elif defined(BP_FAST_PART)
#error "BP_FAST_PART out of range (kFastParts)"
#endif

static_assert(kFastParts == 14, "BP_FAST_LS and the part list must agree");

}  // namespace bp

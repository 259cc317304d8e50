// qb_checks.cuh -- device-side bounds / invariant checks for the checked build
// (-DQB_CHECKS, scripts/gpu_checks.sh).  compute-sanitizer is not available on
// the GPU pool, so the kernels' own index arithmetic is asserted instead: every
// shared-memory list / stack push, every scene / node / pixel index a kernel
// derives at run time.  A failed check prints one line (kernel, file:line,
// block, thread) and the kernel carries on; the checker greps for them.  In the
// production build QB_CHECK compiles to nothing.
#pragma once
#include <cstdio>

#ifdef QB_CHECKS
#define QB_CHECK(cond, what)                                                                                  \
    do {                                                                                                      \
        if (!(cond))                                                                                          \
            printf("QB_CHECK FAILED %s (%s:%d) block %d thread %d\n", what, __FILE__, __LINE__, (int)blockIdx.x, \
                   (int)threadIdx.x);                                                                         \
    } while (0)
#else
#define QB_CHECK(cond, what) \
    do {                     \
    } while (0)
#endif

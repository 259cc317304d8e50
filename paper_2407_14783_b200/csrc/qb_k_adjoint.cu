// qb_k_adjoint.cu -- K1 adjoint (placeholder until the VJP kernel lands).
#include "qb_internal.h"

namespace qb {
int launch_vjp(const qb_params *, int, int, long long, long long, int, const void *, const void *, const void *, void *,
               void *, cudaStream_t) {
    set_error("dynamics adjoint not built yet");
    return QB_EINVAL;
}
}  // namespace qb
